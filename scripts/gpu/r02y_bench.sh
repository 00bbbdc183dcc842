# round 2: bench with the Yahoo leg, smoke(), the C example
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
tail -c 600 gpurun_out/r02y_bench.json; tail -3 gpurun_out/r02y_bench.err
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02y_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02y_smoke.log
tail -3 gpurun_out/r02y_smoke.log
