# round 2: accuracy traces (CTA wavefront lag sources on the Netflix shape; unit grid vs whole blocks on the
# Hugewiki parity slice), the partitioned stream timeline, and the bench with the C4 leg
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/r02e_pytest_wavefront.log 2>&1
tail -5 gpurun_out/r02e_pytest_wavefront.log
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 3 --storage f16,f32 --variants 0,128 --sched wavefront --opt wave_cta=3 > gpurun_out/r02e_wfq_$c.log 2>&1
done
timeout 300 python scripts/probe.py --cfg C2 --epochs 3 --storage f16 --variants 32,64 --sched wavefront > gpurun_out/r02e_warp_wavefront_C2.log 2>&1
timeout 300 python scripts/wavefront_timeline.py --cfg C2 --storage f16 --epochs 2 --wave-cta 0 --variant 64 > gpurun_out/r02e_timeline_warp_C2.log 2>&1
timeout 300 python scripts/wavefront_timeline.py --cfg C2 --storage f16 --epochs 2 --wave-cta 3 > gpurun_out/r02e_timeline_wfq_C2.log 2>&1
cat gpurun_out/r02e_wfq_*.log gpurun_out/r02e_warp_wavefront_C2.log gpurun_out/r02e_timeline_*.log
timeout 900 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 5 \
  --scheds deterministic,hogwild,wavefront,wavefront_cta,wavefront_cta@variant=134217728,wavefront_cta@variant=67108864,wavefront_cta@wave_cta=3 \
  > gpurun_out/r02e_c2_traces.jsonl 2> gpurun_out/r02e_c2_traces.err
timeout 900 python scripts/trace_compare.py --cfg C4-rows10 --storage f32 --epochs 10 \
  --scheds hogwild,partitioned:2:::2,partitioned:4:::2,partitioned:8:::2,partitioned:2:::0,partitioned:4:::0,partitioned:8:::0 \
  > gpurun_out/r02e_c4r10_traces.jsonl 2> gpurun_out/r02e_c4r10_traces.err
timeout 600 python scripts/partition_timeline.py --cfg C4-rows100 --G 4 --modes 0,1,2 > gpurun_out/r02e_timeline_G4.jsonl 2> gpurun_out/r02e_timeline.err
timeout 600 python scripts/partition_timeline.py --cfg C4-rows100 --G 8 --modes 0,2 > gpurun_out/r02e_timeline_G8.jsonl 2>> gpurun_out/r02e_timeline.err
rm -f gpurun_out/partition_timeline_*.json
cat gpurun_out/r02e_*.jsonl
for c in C2 C3; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 3 --storage f16,f32 --variants 0,4194304 --sched deterministic > gpurun_out/r02e_waves_$c.log 2>&1
done
cat gpurun_out/r02e_waves_*.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "deterministic or worked or waves" > gpurun_out/r02e_pytest_waves.log 2>&1
tail -3 gpurun_out/r02e_pytest_waves.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
tail -c 3000 gpurun_out/r02e_bench.json
