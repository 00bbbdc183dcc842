# round 2: after the warp-uniform index fix (no SHFL convergence fix-ups in k_hogwild / k_waves / k_rmse):
# throughput of batch-Hogwild! (register vs TMA-staged triples), deterministic waves, warp-wavefront sizing
set -x
mkdir -p gpurun_out
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --variants 983040,65536 --opt r_staging=1 > gpurun_out/r02i_reg_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --variants 983040,65536 --opt r_staging=2 > gpurun_out/r02i_tma_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 3 --storage f16,f32 --variants 0 --sched deterministic > gpurun_out/r02i_waves_$c.log 2>&1
done
for sc in "2368 2960" "3552 4440" "4736 5920" "3552 7104"; do set -- $sc
  timeout 300 python scripts/probe.py --cfg C2 --epochs 2 --storage f16,f32 --variants 32 --sched wavefront --opt wave_rows=$1 --opt wave_cols=$2 > gpurun_out/r02i_warp_s$1_c$2.log 2>&1
done
timeout 300 python scripts/probe.py --cfg C3 --epochs 2 --storage f16 --variants 32 --sched wavefront --opt wave_rows=2368 --opt wave_cols=2960 > gpurun_out/r02i_warp_C3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02i_pytest_parity.log 2>&1
tail -3 gpurun_out/r02i_pytest_parity.log
cat gpurun_out/r02i_*.log | grep -v "^gen"
