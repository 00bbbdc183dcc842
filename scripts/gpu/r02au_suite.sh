# round 2 (late): flakiness check -- the whole GPU suite again
set -x
mkdir -p gpurun_out
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02au_pytest_gpu.log 2>&1
tail -8 gpurun_out/r02au_pytest_gpu.log
