# round 2: remaining variant sweeps -- batch-Hogwild! fp32 on the Yahoo shape, deterministic fp32 on the Netflix shape
set -x
mkdir -p gpurun_out
timeout 900 python scripts/probe.py --cfg C3 --epochs 4 --storage f32 --variants 0,1,2,16,17,18,32 > gpurun_out/r02bi_hog_C3_f32.log 2>&1
timeout 900 python scripts/probe.py --cfg C2 --epochs 3 --storage f32 --sched deterministic --variants 0,1,2,16777216,16777217,16777218,50331648 > gpurun_out/r02bi_det_C2_f32.log 2>&1
grep -H "G/s" gpurun_out/r02bi_*.log
