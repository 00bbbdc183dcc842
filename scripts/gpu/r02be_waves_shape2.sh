# round 2: deterministic waves on the Yahoo shape -- more shape x form combinations around the 8-lane D = 1 form
set -x
mkdir -p gpurun_out
timeout 900 python scripts/probe.py --cfg C3 --epochs 3 --storage f16 --sched deterministic \
  --variants 16777217,33554433,50331649,16777217,0 > gpurun_out/r02be_waves_C3.log 2>&1
timeout 900 python scripts/probe.py --cfg C3 --epochs 3 --storage f32 --sched deterministic \
  --variants 0,1,16777216,16777217,16777218 > gpurun_out/r02be_waves_C3_f32.log 2>&1
timeout 900 python scripts/probe.py --cfg C3-10pct --epochs 3 --storage f16 --sched deterministic \
  --variants 0,16777217 > gpurun_out/r02be_waves_C3_10pct.log 2>&1
grep -H "G/s" gpurun_out/r02be_*.log
