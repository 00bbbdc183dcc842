# round 2: whole GPU suite + bench with the atomic Q write-back as the batch-Hogwild! default (A-20)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02ab_pytest_gpu.log 2>&1
tail -25 gpurun_out/r02ab_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ab_bench.json 2> gpurun_out/r02ab_bench.err
tail -c 1500 gpurun_out/r02ab_bench.json
