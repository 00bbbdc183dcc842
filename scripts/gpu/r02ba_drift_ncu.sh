# round 2: what changes between an early and a late batch-Hogwild! epoch (ncu metrics of launch 4 vs 30)
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__cycles_elapsed.avg.per_second,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio
for s in 3 29; do
timeout 900 ncu --metrics $M --clock-control none -k regex:k_hogwild -s $s -c 1 --csv --log-file gpurun_out/r02ba_ncu_launch$s.csv \
  python scripts/trace_compare.py --cfg C2 --storage f16 --epochs 31 --scheds hogwild > /dev/null 2>&1
done
ls -la gpurun_out | grep r02ba
