# round 2: out-of-core factors (MF_OPT_P_HOST) parity and errors; a Hugewiki-shaped run with P in pinned host memory
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_outcore.py -q -p no:cacheprovider -rfE > gpurun_out/r02z_pytest_outcore.log 2>&1
tail -15 gpurun_out/r02z_pytest_outcore.log
timeout 1200 python scripts/outcore_c4.py > gpurun_out/r02z_outcore_c4.json 2> gpurun_out/r02z_outcore_c4.err
cat gpurun_out/r02z_outcore_c4.json; tail -3 gpurun_out/r02z_outcore_c4.err
