# round 2: the Zipf slice, partitioned G = 4 -- passes per epoch and workers per partition
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2-zipf-1pct --storage f32 --epochs 10 \
  --scheds partitioned:4,partitioned:4:8,partitioned:4:16,partitioned:4:32,partitioned:4:4:1,partitioned:4:16:1,partitioned:4:4:4,partitioned:4:8:4,partitioned:4:4::0,partitioned:4:16::0,partitioned:2,partitioned:8 \
  > gpurun_out/r02ag_zipf_part.jsonl 2> gpurun_out/r02ag_zipf_part.err
tail -c 300 gpurun_out/r02ag_zipf_part.err
