# round 2: deterministic waves with an L2 prefetch of the next wave's first-step rows before the barrier
# (MF_OPT_VARIANT bits 16..19 = 1) vs without; the kappa test and the waves' bitwise test
set -x
mkdir -p gpurun_out
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --sched deterministic --variants 0,65536,0,65536 > gpurun_out/r02aj_waves_$c.log 2>&1
done
grep -h "G/s" gpurun_out/r02aj_waves_*.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "kappa or bitwise" > gpurun_out/r02aj_pytest.log 2>&1
tail -3 gpurun_out/r02aj_pytest.log
