# round 2: CTA wavefront on the Netflix shape with its 3 passes -- in-block clamp (bits 26..27) and shape (bits 8..11)
set -x
mkdir -p gpurun_out
for s in f16 f32; do
timeout 900 python scripts/probe.py --cfg C2 --epochs 4 --storage $s --sched wavefront --opt wave_cta=1 \
  --variants 0,67108864,134217728,201326592,256,512,0 > gpurun_out/r02bj_cta_C2_$s.log 2>&1
done
grep -H "G/s" gpurun_out/r02bj_*.log
