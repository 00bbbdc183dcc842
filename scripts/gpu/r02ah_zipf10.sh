# round 2: the 10% Zipf slice (C2-zipf-10pct), every schedule, 10 epochs, fp32 and fp16
set -x
mkdir -p gpurun_out
for s in f32 f16; do
timeout 1200 python scripts/trace_compare.py --cfg C2-zipf-10pct --storage $s --epochs 10 \
  --scheds deterministic,hogwild,wavefront_cta,wavefront,partitioned:2,partitioned:4,partitioned:8 \
  > gpurun_out/r02ah_zipf10_$s.jsonl 2> gpurun_out/r02ah_zipf10_$s.err
tail -c 300 gpurun_out/r02ah_zipf10_$s.err
done
