# round 2: deterministic dataflow execution (per-row counters, no barriers) + auto Q write-back by kappa
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "deterministic or degenerate or worked or q_store" > gpurun_out/r02ac_pytest_det.log 2>&1
tail -5 gpurun_out/r02ac_pytest_det.log
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --sched deterministic --opt det_flow=1 > gpurun_out/r02ac_flow_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16 --sched hogwild > gpurun_out/r02ac_hog_$c.log 2>&1
done
grep -h "G/s" gpurun_out/r02ac_flow_*.log gpurun_out/r02ac_hog_*.log
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02ac_pytest_gpu.log 2>&1
tail -25 gpurun_out/r02ac_pytest_gpu.log
