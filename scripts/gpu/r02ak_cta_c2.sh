# round 2: CTA wavefront on the fp16 Netflix trace -- in-block clamp and pass count vs the late-epoch drift
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 \
  --scheds wavefront_cta,wavefront_cta@variant=67108864,wavefront_cta@variant=134217728,wavefront_cta@wave_passes=3,wavefront_cta@wave_passes=4,hogwild \
  > gpurun_out/r02ak_c2_f16.jsonl 2> gpurun_out/r02ak_c2_f16.err
tail -c 300 gpurun_out/r02ak_c2_f16.err
