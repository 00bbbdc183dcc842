# round 2: Q write-back as an atomic add of the change (MF_OPT_Q_UPDATE) -- throughput and accuracy vs store
set -x
mkdir -p gpurun_out
for c in C2 C3; do
  for q in 0 1; do
    timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16,f32 --opt q_update=$q > gpurun_out/r02aa_probe_${c}_q$q.log 2>&1
  done
done
grep -h "" gpurun_out/r02aa_probe_*.log | tail -40
for s in f16 f32; do
  timeout 900 python scripts/trace_compare.py --cfg C4-rows100 --storage $s --epochs 20 \
    --scheds hogwild@q_update=1,partitioned:2@q_update=1,partitioned:4@q_update=1,partitioned:8@q_update=1,hogwild@q_update=0 \
    > gpurun_out/r02aa_c4r100_$s.jsonl 2> gpurun_out/r02aa_c4r100_$s.err
done
timeout 900 python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 20 --scheds hogwild@q_update=1 \
    > gpurun_out/r02aa_c2_f16.jsonl 2> gpurun_out/r02aa_c2_f16.err
timeout 900 python scripts/trace_compare.py --cfg C4-rows10 --storage f16 --epochs 10 \
    --scheds hogwild@q_update=1,partitioned:4@q_update=1 > gpurun_out/r02aa_c4r10_f16.jsonl 2> gpurun_out/r02aa_c4r10_f16.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -x -q -p no:cacheprovider > gpurun_out/r02aa_pytest.log 2>&1
tail -5 gpurun_out/r02aa_pytest.log
