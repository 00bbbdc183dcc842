# round 2: the Zipf slice -- paper-literal wavefront passes, partitioned Q write-back forms
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2-zipf-1pct --storage f32 --epochs 10 \
  --scheds deterministic,wavefront,wavefront@wave_passes=2,wavefront@wave_passes=4,wavefront@wave_passes=8,wavefront@wave_passes=16,wavefront_cta,partitioned:4,partitioned:4@q_update=1,hogwild,hogwild@q_update=1 \
  > gpurun_out/r02af_zipf.jsonl 2> gpurun_out/r02af_zipf.err
tail -c 800 gpurun_out/r02af_zipf.err
