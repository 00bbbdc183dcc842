# round 2: the multi-GPU bench path as the driver launches it, on the one GPU a box has: torchrun with one
# rank (real NCCL, the default BASELINE configs[3] workload -- the whole Hugewiki shape on one rank, unit
# grid), and the fake-NCCL multi-rank tests
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.used,memory.total --format=csv > gpurun_out/r02l_mem.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --partitioned --steps 5 --warmup 3 > gpurun_out/r02l_bench_partitioned_C4.json 2> gpurun_out/r02l_bench_partitioned_C4.err
tail -c 2500 gpurun_out/r02l_bench_partitioned_C4.json
tail -5 gpurun_out/r02l_bench_partitioned_C4.err
timeout 900 python -m pytest tests/test_gpu_bench_multirank.py tests/test_gpu_nccl_fake.py tests/test_gpu_partition.py -q -p no:cacheprovider > gpurun_out/r02l_pytest_multi.log 2>&1
tail -3 gpurun_out/r02l_pytest_multi.log
