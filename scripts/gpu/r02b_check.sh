# round 2: suite + bench on the current HEAD (after the L2 evict_first / footprint commit)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02b_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
tail -c 1500 gpurun_out/r02b_bench.json
