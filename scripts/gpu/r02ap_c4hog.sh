# round 2: batch-Hogwild! on the full Hugewiki shape -- ratings in flight per warp, L2 prefetch, Q write-back
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/probe.py --cfg C4 --epochs 3 --storage f16 --variants 983040,983072,983104,65536,1 > gpurun_out/r02ap_c4_hog.log 2>&1
timeout 900 python scripts/probe.py --cfg C4 --epochs 3 --storage f16 --variants 983040 --opt q_update=0 > gpurun_out/r02ap_c4_hog_store.log 2>&1
grep -h "G/s" gpurun_out/r02ap_c4_hog*.log
