# round 2: deterministic waves, 512-thread CTAs x 2 per SM with 4 samples per group (bits 24..25 = 3)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "deterministic" > gpurun_out/r02t_pytest.log 2>&1
tail -3 gpurun_out/r02t_pytest.log
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 3 --storage f16,f32 --variants 0,50331648 --sched deterministic > gpurun_out/r02t_waves_$c.log 2>&1
done
cat gpurun_out/r02t_waves_*.log | grep -v "^gen"
timeout 1200 python -m pytest tests/test_gpu_wavefront.py -q -p no:cacheprovider > gpurun_out/r02t_pytest_wavefront.log 2>&1
tail -3 gpurun_out/r02t_pytest_wavefront.log
