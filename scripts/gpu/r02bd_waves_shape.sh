# round 2: deterministic waves on the Yahoo shape -- group shape (bits 0..3) x samples per group (bits 24..25)
set -x
mkdir -p gpurun_out
timeout 900 python scripts/probe.py --cfg C3 --epochs 3 --storage f16 --sched deterministic \
  --variants 0,1,2,3,16777216,16777217,16777218,16777219,50331648,50331650 > gpurun_out/r02bd_waves_C3.log 2>&1
timeout 900 python scripts/probe.py --cfg C2 --epochs 3 --storage f16 --sched deterministic \
  --variants 0,1,2,3,16777218 > gpurun_out/r02bd_waves_C2.log 2>&1
grep -H "G/s" gpurun_out/r02bd_*.log
