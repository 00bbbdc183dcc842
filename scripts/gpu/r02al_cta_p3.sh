# round 2: CTA wavefront auto passes round(sqrt(V / 5)) -- the wavefront tests, the full-size traces, the bench
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_wavefront.py tests/test_gpu_slices.py -q -p no:cacheprovider -rfEx -k "wavefront or cta" > gpurun_out/r02al_pytest.log 2>&1
tail -8 gpurun_out/r02al_pytest.log
timeout 1200 python scripts/trace_compare.py --cfg C2 --storage f32 --epochs 20 --scheds wavefront_cta > gpurun_out/r02al_c2_f32.jsonl 2> gpurun_out/r02al_c2_f32.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02al_bench.json 2> gpurun_out/r02al_bench.err
tail -c 600 gpurun_out/r02al_bench.json
