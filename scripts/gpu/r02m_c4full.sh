# round 2: the whole Hugewiki shape (3.07 B ratings) on one GPU: per-epoch test RMSE of exact serial SGD
# (deterministic waves), batch-Hogwild! and the partitioned schedule with G = 2 / 4 / 8 loopback partitions
# (the same per-partition worker counts and order as G GPUs), fp16; plus the sanitizer over every kernel family
set -x
mkdir -p gpurun_out
timeout 2400 python scripts/trace_compare.py --cfg C4 --storage f16 --epochs 10 --shuffle 0 \
  --scheds hogwild,partitioned:8,partitioned:4,partitioned:2,deterministic > gpurun_out/r02m_c4_traces.jsonl 2> gpurun_out/r02m_c4_traces.err
cat gpurun_out/r02m_c4_traces.jsonl
tail -3 gpurun_out/r02m_c4_traces.err
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_run.py > gpurun_out/r02m_sanitizer.log 2>&1; echo "sanitizer rc=$?" >> gpurun_out/r02m_sanitizer.log
tail -5 gpurun_out/r02m_sanitizer.log
