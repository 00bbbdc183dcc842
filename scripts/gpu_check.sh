#!/bin/bash
# One GPU round trip: smoke, gpu tests, bench, launch list, ncu capture of the update kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
  cat gpurun_out/bench_f16.json
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-variants --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
  mkdir -p /tmp/ncu
  for st in f16 f32; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hogwild -s 3 -c 1 \
       -o /tmp/ncu/prof_hogwild_$st -f python bench.py --storage $st --steps 1 --warmup 3 --no-cpu --no-variants --e2e-steps 1 > gpurun_out/ncu_full_$st.log 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wavefront_cta -s 3 -c 1 \
       -o /tmp/ncu/prof_wfcta_$st -f python bench.py --storage $st --schedule wavefront_cta --steps 1 --warmup 3 --no-cpu --no-variants --e2e-steps 1 > gpurun_out/ncu_wfcta_$st.log 2>&1
  done
  # raw metric pages travel back (the .ncu-rep files together exceed gpurun's 64 MiB copy-back)
  for f in /tmp/ncu/*.ncu-rep; do
    b=$(basename $f .ncu-rep)
    ncu -i $f --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
    ncu -i $f --page source --csv > gpurun_out/$b.source.csv 2>/dev/null
  done
  cp /tmp/ncu/prof_hogwild_f16.ncu-rep gpurun_out/ 2>/dev/null
fi
ls gpurun_out
