# round 2: ncu evidence for the final defaults -- the launch list of the bench command, a full capture of the
# headline kernel, per-config DRAM bytes of the new batch-Hogwild! default shapes
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02u_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-variants --no-c4 --no-cpu --e2e-steps 1 > gpurun_out/r02u_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_hogwild -s 4 -c 1 -o gpurun_out/r02u_hogwild_C2_f16 \
  python scripts/probe.py --cfg C2 --epochs 6 --storage f16 --variants -1 > gpurun_out/r02u_full.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
for spec in "C2 f16" "C2 f32" "C3 f16" "C3 f32" "C4 f16"; do set -- $spec
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_hogwild -s 4 -c 1 --csv --log-file gpurun_out/r02u_ncu_$1_$2_hogwild.csv \
    python scripts/probe.py --cfg $1 --epochs 6 --storage $2 --variants -1 > /dev/null 2>&1
done
timeout 900 ncu --metrics $M --clock-control none -k regex:k_wavefront_cta -s 4 -c 1 --csv --log-file gpurun_out/r02u_ncu_C4_f16_wavefront.csv \
    python scripts/probe.py --cfg C4 --epochs 6 --storage f16 --variants -1 --sched wavefront --opt wave_cta=1 > /dev/null 2>&1
ls -la gpurun_out | grep r02u
