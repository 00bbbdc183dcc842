# round 2 (late): compute-sanitizer memcheck over every kernel family, incl. the atomic Q write-back and k_flow
set -x
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_run.py > gpurun_out/r02am_sanitizer.log 2>&1; echo "sanitizer rc=$?" >> gpurun_out/r02am_sanitizer.log
tail -5 gpurun_out/r02am_sanitizer.log
