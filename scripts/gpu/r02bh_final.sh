# round 2 final (after the large-wave form and the chunk default): GPU suite, smoke, bench as the driver runs it
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02bh_pytest_gpu.log 2>&1
tail -8 gpurun_out/r02bh_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bh_smoke.log 2>&1
tail -1 gpurun_out/r02bh_smoke.log
timeout 1200 python bench.py > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err
tail -c 800 gpurun_out/r02bh_bench.json
