set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
python scripts/probe.py --cfg C2 --epochs 4 --storage f16,f32 --variants 983040,269418496,537853952,806289408 > gpurun_out/r02a_policy_C2.log 2>&1
python scripts/probe.py --cfg C3 --epochs 4 --storage f16 --variants 983040,269418496,537853952,806289408,0 > gpurun_out/r02a_policy_C3.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_hogwild --csv --log-file gpurun_out/r02a_ncu_policy_C2.csv python scripts/probe.py --cfg C2 --epochs 2 --storage f16 --variants 983040,269418496,537853952,806289408 > gpurun_out/r02a_ncu_probe.log 2>&1
cat gpurun_out/r02a_policy_C2.log gpurun_out/r02a_policy_C3.log
