# round 2: the L2 ceilings (stream / random-row RMW) with ncu naming the saturated unit, the update
# pattern's ceiling under ncu, and per-config DRAM traffic of the update kernels (C2, C3, C4)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/r02d_pytest_wavefront.log 2>&1
tail -3 gpurun_out/r02d_pytest_wavefront.log
for c in "C2 f16,f32" "C3 f16"; do set -- $c
  timeout 600 python scripts/probe.py --cfg $1 --epochs 3 --storage $2 --variants 32,64,128 --sched wavefront > gpurun_out/r02d_warp_wavefront_$1.log 2>&1
done
cat gpurun_out/r02d_warp_wavefront_*.log
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo"
$NV -o /tmp/l2c scripts/l2_ceiling.cu && $NV -o /tmp/smc scripts/sgd_mem_ceiling.cu
timeout 300 /tmp/l2c > gpurun_out/r02d_l2_ceiling.jsonl 2>&1
M=gpu__time_duration.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_l1tex2xbar_write_bytes.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,lts__d_sectors.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02d_ncu_l2_ceiling.csv /tmp/l2c 48 > gpurun_out/r02d_l2c48.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:rmw -s 1 -c 1 -o gpurun_out/r02d_smc_C2_f16 /tmp/smc 480190 17771 99072112 256 0 32 1 > gpurun_out/r02d_smc.log 2>&1
for spec in "C2 f16 hogwild" "C2 f32 hogwild" "C2 f16 wavefront" "C3 f16 hogwild" "C3 f32 hogwild" "C3 f16 wavefront" "C4 f16 hogwild" "C4 f16 wavefront"; do
  set -- $spec
  K=k_hogwild; OPT=""; if [ $3 = wavefront ]; then K=k_wavefront_cta; OPT="--opt wave_cta=1"; fi
  timeout 900 ncu --metrics $M --clock-control none -k regex:$K -s 4 -c 1 --csv --log-file gpurun_out/r02d_ncu_$1_$2_$3.csv \
    python scripts/probe.py --cfg $1 --epochs 6 --storage $2 --variants 0 --sched $3 $OPT > gpurun_out/r02d_probe_$1_$2_$3.log 2>&1
done
ls -la gpurun_out
