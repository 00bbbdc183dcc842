# round 2: deterministic dataflow, round-robin ownership (forms: 0 = 64 regs, 1 = 40, 3 = 32) vs the waves
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "deterministic or degenerate or worked" > gpurun_out/r02ad_pytest_det.log 2>&1
tail -3 gpurun_out/r02ad_pytest_det.log
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --sched deterministic --opt det_flow=1 --variants 0,16777216,50331648 > gpurun_out/r02ad_flow_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --sched deterministic --opt det_flow=0 > gpurun_out/r02ad_waves_$c.log 2>&1
done
grep -h "G/s" gpurun_out/r02ad_*.log
