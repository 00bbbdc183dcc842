# round 2: CTA wavefront with 2 / 4 passes on the Netflix shape (20 epochs, both storages) and the Yahoo shape
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 \
  --scheds wavefront_cta@wave_passes=2,wavefront_cta@wave_passes=4,wavefront > gpurun_out/r02v_c2_f16.jsonl 2> gpurun_out/r02v.err
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f32 --epochs 20 \
  --scheds wavefront_cta,wavefront_cta@wave_passes=2 > gpurun_out/r02v_c2_f32.jsonl 2>> gpurun_out/r02v.err
timeout 1200 python scripts/trace_compare.py --cfg C3 --storage f16 --epochs 6 \
  --scheds wavefront_cta@wave_passes=2,hogwild,deterministic > gpurun_out/r02v_c3_f16.jsonl 2>> gpurun_out/r02v.err
cat gpurun_out/r02v_*.jsonl | cut -c1-300
