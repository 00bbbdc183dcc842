# round 2: batch-Hogwild! 8-lane shape (variant 1) vs the 32-lane default where P does not fit L2
set -x
mkdir -p gpurun_out
timeout 900 python scripts/probe.py --cfg C3 --epochs 4 --storage f16 --variants 0,1,983040,983041,0,1 > gpurun_out/r02aq_c3.log 2>&1
timeout 900 python scripts/probe.py --cfg C4-rows10 --epochs 4 --storage f16 --variants 0,1,0,1 > gpurun_out/r02aq_c4r10.log 2>&1
timeout 1500 python scripts/probe.py --cfg C4 --epochs 4 --storage f16 --variants 0,1 --sched partitioned --opt partitions=1 > gpurun_out/r02aq_c4_part.log 2>&1
grep -h "G/s" gpurun_out/r02aq_*.log
