# round 2: CTA wavefront group shapes (bits 8..11) and ratings in flight per group (bits 12..15) on the
# Yahoo and Hugewiki-rows/10 shapes; warp-wavefront depth (bits 4..7) on the Yahoo shape
set -x
mkdir -p gpurun_out
for c in C3 C4-rows10; do
  timeout 900 python scripts/probe.py --cfg $c --epochs 4 --storage f16 --sched wavefront --opt wave_cta=1 \
    --variants 0,256,512,768,1024,4096,8192,4352,4608 > gpurun_out/r02bg_cta_${c}_f16.log 2>&1
  timeout 900 python scripts/probe.py --cfg $c --epochs 4 --storage f32 --sched wavefront --opt wave_cta=1 \
    --variants 0,256,512,768,1024,4096,8192 > gpurun_out/r02bg_cta_${c}_f32.log 2>&1
done
timeout 900 python scripts/probe.py --cfg C3 --epochs 3 --storage f16 --sched wavefront --variants 0,32,64,128 > gpurun_out/r02bg_warp_C3.log 2>&1
grep -H "G/s" gpurun_out/r02bg_*.log
