# round 2 (late): ncu --set full of the CTA wavefront launch (Yahoo and Netflix shapes, fp16, current defaults)
set -x
mkdir -p gpurun_out
for c in C3 C2; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_wavefront_cta -s 4 -c 1 -o gpurun_out/r02at_wfcta_${c}_f16 \
  python scripts/probe.py --cfg $c --epochs 6 --storage f16 --variants -1 --sched wavefront --opt wave_cta=1 > gpurun_out/r02at_full_$c.log 2>&1
done
ls -la gpurun_out | grep r02at
