# round 2: per-epoch test RMSE + kernel time of every single-GPU schedule (time to serial SGD's RMSE);
# CTA wavefront q_v read late (default) vs early (MF_OPT_VARIANT bit 22)
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 \
  --scheds deterministic,hogwild,wavefront_cta,wavefront_cta@variant=4194304,wavefront \
  > gpurun_out/r02ae_c2_f16.jsonl 2> gpurun_out/r02ae_c2_f16.err
timeout 1200 python scripts/trace_compare.py --cfg C3 --storage f16 --epochs 10 \
  --scheds deterministic,hogwild,wavefront_cta,wavefront_cta@variant=4194304,wavefront \
  > gpurun_out/r02ae_c3_f16.jsonl 2> gpurun_out/r02ae_c3_f16.err
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f32 --epochs 20 \
  --scheds deterministic,hogwild,wavefront_cta,wavefront \
  > gpurun_out/r02ae_c2_f32.jsonl 2> gpurun_out/r02ae_c2_f32.err
tail -c 600 gpurun_out/r02ae_c2_f16.err
