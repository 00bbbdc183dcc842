# round 2: deterministic waves, auto large-wave form -- full-size Yahoo parity (fp32 / fp16) and throughput
set -x
mkdir -p gpurun_out
timeout 600 python scripts/probe.py --cfg C3 --epochs 3 --storage f16,f32 --sched deterministic --variants 0 > gpurun_out/r02bf_probe_C3.log 2>&1
timeout 600 python scripts/probe.py --cfg C2 --epochs 3 --storage f16 --sched deterministic --variants 0 > gpurun_out/r02bf_probe_C2.log 2>&1
grep -h "G/s" gpurun_out/r02bf_probe_*.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_slices.py -q -p no:cacheprovider -rfEx -k "c3 or deterministic or C3" > gpurun_out/r02bf_pytest.log 2>&1
tail -6 gpurun_out/r02bf_pytest.log
