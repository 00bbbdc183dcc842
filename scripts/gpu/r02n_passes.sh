# round 2: what closes the partitioned schedule's lag on the Hugewiki parity slice (C4-rows100): more passes
# per epoch (S), fewer workers per partition
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/trace_compare.py --cfg C4-rows100 --storage f16 --epochs 20 \
  --scheds partitioned:4:8,partitioned:4:16,partitioned:8:16,partitioned:8:32,partitioned:4:4:768,hogwild@workers=1536 > gpurun_out/r02n_c4r100_f16.jsonl 2> gpurun_out/r02n.err
timeout 1500 python scripts/trace_compare.py --cfg C4-rows100 --storage f32 --epochs 20 \
  --scheds partitioned:4:8,partitioned:4:16,partitioned:8:16,partitioned:8:32 > gpurun_out/r02n_c4r100_f32.jsonl 2>> gpurun_out/r02n.err
tail -3 gpurun_out/r02n.err
timeout 2400 python scripts/trace_compare.py --cfg C4 --storage f16 --epochs 6 --shuffle 0 \
  --scheds partitioned:2:40,partitioned:4:20,partitioned:8:10,partitioned:8:20 > gpurun_out/r02n_c4_f16.jsonl 2>> gpurun_out/r02n.err
cat gpurun_out/r02n_*.jsonl
