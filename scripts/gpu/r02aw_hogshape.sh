# round 2: batch-Hogwild! auto shape (8-lane where P >> L2 and Q << L2) -- throughput and the Hugewiki parity gates
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/probe.py --cfg C4 --epochs 4 --storage f16 --variants 0,2,0,2 > gpurun_out/r02aw_c4.log 2>&1
timeout 900 python scripts/probe.py --cfg C4-rows10 --epochs 4 --storage f16 --variants 0,2,0,2 > gpurun_out/r02aw_c4r10.log 2>&1
timeout 900 python scripts/probe.py --cfg C2 --epochs 4 --storage f16 --variants 0,2 > gpurun_out/r02aw_c2.log 2>&1
timeout 900 python scripts/probe.py --cfg C3 --epochs 4 --storage f16 --variants 0,2 > gpurun_out/r02aw_c3.log 2>&1
grep -H "G/s" gpurun_out/r02aw_*.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -rfEx -k "c4" > gpurun_out/r02aw_pytest.log 2>&1
tail -6 gpurun_out/r02aw_pytest.log
