# round 2 (late): GPU suite, bench, smoke, ncu launch list of the bench, full capture of the headline kernel,
# per-config DRAM bytes of the batch-Hogwild! launches (C3 / C4 now take the atomic Q write-back, A-20)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02ai_pytest_gpu.log 2>&1
tail -12 gpurun_out/r02ai_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ai_smoke.log 2>&1
tail -2 gpurun_out/r02ai_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ai_bench.json 2> gpurun_out/r02ai_bench.err
tail -c 1200 gpurun_out/r02ai_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02ai_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-variants --no-c4 --no-cpu --e2e-steps 1 > gpurun_out/r02ai_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_hogwild -s 4 -c 1 -o gpurun_out/r02ai_hogwild_C2_f16 \
  python scripts/probe.py --cfg C2 --epochs 6 --storage f16 --variants -1 > gpurun_out/r02ai_full.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
for spec in "C3 f16" "C3 f32" "C4 f16"; do set -- $spec
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_hogwild -s 4 -c 1 --csv --log-file gpurun_out/r02ai_ncu_$1_$2_hogwild.csv \
    python scripts/probe.py --cfg $1 --epochs 6 --storage $2 --variants -1 > /dev/null 2>&1
done
ls -la gpurun_out | grep r02ai
