# round 2: CTA wavefront column groups c vs workers s = 148 with 2 passes (Netflix shape): block-boundary cost
set -x
mkdir -p gpurun_out
for c in 148 164 185 222; do
  timeout 300 python scripts/probe.py --cfg C2 --epochs 4 --storage f16,f32 --variants 0 --sched wavefront --opt wave_cta=1 --opt wave_passes=2 --opt wave_cols=$c > gpurun_out/r02x_c$c.log 2>&1
done
timeout 300 python scripts/wavefront_timeline.py --cfg C2 --storage f16 --epochs 2 --wave-cta 1 > gpurun_out/r02x_timeline_p2.log 2>&1
timeout 600 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 5 --scheds wavefront_cta@wave_cols=185,wavefront_cta@wave_cols=222 > gpurun_out/r02x_traces.jsonl 2>&1
cat gpurun_out/r02x_c*.log | grep -v "^gen"; cat gpurun_out/r02x_timeline_p2.log gpurun_out/r02x_traces.jsonl
