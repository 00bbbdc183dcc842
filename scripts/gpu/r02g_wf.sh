# round 2: the wavefront kernels without convergence fix-ups around their shuffles
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavefront.py -q -p no:cacheprovider > gpurun_out/r02g_pytest_wavefront.log 2>&1
tail -5 gpurun_out/r02g_pytest_wavefront.log
timeout 600 python scripts/probe.py --cfg C2 --epochs 3 --storage f16,f32 --variants 32,64,128 --sched wavefront > gpurun_out/r02g_warp_C2.log 2>&1
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 3 --storage f16,f32 --variants 0,128,32 --sched wavefront --opt wave_cta=3 > gpurun_out/r02g_wfq_$c.log 2>&1
done
timeout 300 python scripts/wavefront_timeline.py --cfg C2 --storage f16 --epochs 2 --wave-cta 0 --variant 64 > gpurun_out/r02g_timeline_warp_C2.log 2>&1
cat gpurun_out/r02g_warp_C2.log gpurun_out/r02g_wfq_*.log gpurun_out/r02g_timeline_warp_C2.log
