# round 2: TMA-staged triples for batch-Hogwild! (parity + throughput), warp-wavefront sizing sweep
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tma or worked or exactly" > gpurun_out/r02h_pytest_tma.log 2>&1
tail -5 gpurun_out/r02h_pytest_tma.log
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --variants 983040,65536 --opt r_staging=1 > gpurun_out/r02h_reg_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --variants 983040,65536 --opt r_staging=2 > gpurun_out/r02h_tma_$c.log 2>&1
done
for sc in "1184 1480" "1184 2368" "2368 2960" "2368 4736" "1776 2220" "1776 3552"; do set -- $sc
  timeout 300 python scripts/probe.py --cfg C2 --epochs 2 --storage f16 --variants 32 --sched wavefront --opt wave_rows=$1 --opt wave_cols=$2 > gpurun_out/r02h_warp_s$1_c$2.log 2>&1
done
cat gpurun_out/r02h_reg_*.log gpurun_out/r02h_tma_*.log gpurun_out/r02h_warp_*.log
