# round 2: wavefront passes (fresh column sequences per 1/P of the samples): parity tests, accuracy and
# throughput on the Netflix and Hugewiki shapes
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wavefront.py -q -p no:cacheprovider > gpurun_out/r02r_pytest_wavefront.log 2>&1
tail -3 gpurun_out/r02r_pytest_wavefront.log
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 5 \
  --scheds wavefront_cta@wave_passes=4,wavefront_cta@wave_passes=16,wavefront@wave_passes=4,wavefront_cta@wave_passes=4@wave_cta=3 > gpurun_out/r02r_c2.jsonl 2> gpurun_out/r02r.err
timeout 2400 python scripts/trace_compare.py --cfg C4 --storage f16 --epochs 5 --shuffle 0 \
  --scheds wavefront_cta@wave_passes=8,wavefront_cta@wave_passes=32,wavefront_cta@wave_passes=128,wavefront@wave_passes=8 > gpurun_out/r02r_c4.jsonl 2>> gpurun_out/r02r.err
cat gpurun_out/r02r_*.jsonl; tail -3 gpurun_out/r02r.err
