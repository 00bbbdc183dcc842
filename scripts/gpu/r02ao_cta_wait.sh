# round 2: CTA wavefront, Q-group copy-in waited at the first rating (default) vs before the tile claims (bit 23)
set -x
mkdir -p gpurun_out
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --sched wavefront --opt wave_cta=1 --variants 0,8388608,0,8388608 > gpurun_out/r02ao_cta_$c.log 2>&1
done
grep -h "G/s" gpurun_out/r02ao_cta_*.log
timeout 1200 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/r02ao_pytest.log 2>&1
tail -3 gpurun_out/r02ao_pytest.log
