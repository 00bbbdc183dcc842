# round 2: CTA wavefront, one 1024-thread worker per SM vs two 512-thread workers (MF_OPT_WAVE_CTA = 2)
set -x
mkdir -p gpurun_out
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16 --sched wavefront --opt wave_cta=1 --variants 0,0 > gpurun_out/r02as_cta1_$c.log 2>&1
  timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16 --sched wavefront --opt wave_cta=2 --variants 0,0 > gpurun_out/r02as_cta2_$c.log 2>&1
done
grep -H "G/s" gpurun_out/r02as_*.log
timeout 900 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 --scheds wavefront_cta@wave_cta=2 > gpurun_out/r02as_c2_trace.jsonl 2>&1
