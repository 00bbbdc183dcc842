# round 2: the whole GPU suite and the bench after the auto pass count, slice tests and full-size C4 test
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02o_pytest_gpu.log 2>&1
tail -30 gpurun_out/r02o_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
tail -c 1200 gpurun_out/r02o_bench.json
