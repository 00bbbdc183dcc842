# round 2: run-to-run spread of the CTA wavefront's fp16 Netflix trace (3 passes, auto)
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 \
  --scheds wavefront_cta,wavefront_cta,wavefront_cta,wavefront_cta,wavefront_cta,hogwild,hogwild,hogwild \
  > gpurun_out/r02ar_c2_f16_rep.jsonl 2> gpurun_out/r02ar.err
tail -c 300 gpurun_out/r02ar.err
