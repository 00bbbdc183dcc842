# round 2 (late): GPU suite, smoke, bench after the CTA pass rule; ncu DRAM bytes of the CTA wavefront (3 passes)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider -rfEx > gpurun_out/r02an_pytest_gpu.log 2>&1
tail -8 gpurun_out/r02an_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02an_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02an_bench.json 2> gpurun_out/r02an_bench.err
tail -c 600 gpurun_out/r02an_bench.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
for spec in "C2 f16" "C2 f32"; do set -- $spec
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_wavefront_cta -s 4 -c 1 --csv --log-file gpurun_out/r02an_ncu_$1_$2_wfcta.csv \
    python scripts/probe.py --cfg $1 --epochs 6 --storage $2 --variants -1 --sched wavefront --opt wave_cta=1 > /dev/null 2>&1
done
ls -la gpurun_out | grep r02an
