# round 2: unit-grid partition (MF_OPT_PART_SPLIT = 2) parity + accuracy, then the whole suite and bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_nccl_fake.py -x -q -p no:cacheprovider > gpurun_out/r02c_partition.log 2>&1
tail -3 gpurun_out/r02c_partition.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -k c4_rows10 -q -p no:cacheprovider -rA > gpurun_out/r02c_c4rows10.log 2>&1
tail -15 gpurun_out/r02c_c4rows10.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/r02c_pytest_gpu.log 2>&1
tail -5 gpurun_out/r02c_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
tail -c 1500 gpurun_out/r02c_bench.json
