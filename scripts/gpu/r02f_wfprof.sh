# round 2: ncu source-level captures of the two slow wavefront forms (warp workers, q-stationary CTA) on the
# 10% Netflix slice, to see where the in-block time per sample goes
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wavefront -s 1 -c 1 -o gpurun_out/r02f_warp_wf \
  python scripts/probe.py --cfg C2-10pct --epochs 2 --storage f16 --variants 64 --sched wavefront > gpurun_out/r02f_warp.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wavefront_q -s 1 -c 1 -o gpurun_out/r02f_wfq \
  python scripts/probe.py --cfg C2-10pct --epochs 2 --storage f16 --variants 0 --sched wavefront --opt wave_cta=3 > gpurun_out/r02f_wfq.log 2>&1
timeout 600 python scripts/probe.py --cfg C2 --epochs 3 --storage f16,f32 --variants 983040,1074724864,1343160320,1611595776,1880031232 > gpurun_out/r02f_policy_C2.log 2>&1
cat gpurun_out/r02f_policy_C2.log
ls -la gpurun_out | grep r02f
