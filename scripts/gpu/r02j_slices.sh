# round 2: per-epoch test RMSE of every schedule on the fp16 parity slices (C3-10pct, C4-rows100) and
# C4-rows100 fp32, against the oracle goldens (tests/golden/*_trace.json)
set -x
mkdir -p gpurun_out
timeout 900 python scripts/trace_compare.py --cfg C3-10pct --storage f16 --epochs 10 \
  --scheds hogwild,wavefront_cta,wavefront,deterministic > gpurun_out/r02j_c3_10pct_f16.jsonl 2> gpurun_out/r02j.err
timeout 1200 python scripts/trace_compare.py --cfg C4-rows100 --storage f16 --epochs 20 \
  --scheds hogwild,partitioned:2,partitioned:4,partitioned:8,wavefront_cta,deterministic > gpurun_out/r02j_c4_rows100_f16.jsonl 2>> gpurun_out/r02j.err
timeout 1200 python scripts/trace_compare.py --cfg C4-rows100 --storage f32 --epochs 20 \
  --scheds hogwild,partitioned:2,partitioned:4,partitioned:8,deterministic > gpurun_out/r02j_c4_rows100_f32.jsonl 2>> gpurun_out/r02j.err
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 \
  --scheds hogwild,wavefront_cta > gpurun_out/r02j_c2_f16.jsonl 2>> gpurun_out/r02j.err
tail -3 gpurun_out/r02j.err
timeout 900 python -m pytest tests/test_gpu_wavefront.py -q -p no:cacheprovider > gpurun_out/r02j_pytest_wavefront.log 2>&1
tail -3 gpurun_out/r02j_pytest_wavefront.log
timeout 300 python scripts/probe.py --cfg C2 --epochs 3 --storage f16,f32 --variants 0,32 --sched wavefront > gpurun_out/r02j_warp_C2.log 2>&1
timeout 300 python scripts/probe.py --cfg C2 --epochs 4 --storage f16,f32 --variants 983040 > gpurun_out/r02j_hog_C2.log 2>&1
cat gpurun_out/r02j_warp_C2.log gpurun_out/r02j_hog_C2.log
