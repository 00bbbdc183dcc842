# round 2: C5, the k sweep on the Netflix shape (k = 32 / 64 / 128 / 256, fp16 and fp32): throughput of
# batch-Hogwild!, the CTA wavefront and the warp wavefront, and ncu DRAM / L2 bytes of the batch-Hogwild!
# launch per (k, storage)
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
for k in 32 64 128 256; do
  timeout 600 python scripts/probe.py --cfg C2 --k $k --epochs 4 --storage f16,f32 --variants 983040 > gpurun_out/r02k_hog_k$k.log 2>&1
  timeout 600 python scripts/probe.py --cfg C2 --k $k --epochs 4 --storage f16,f32 --variants 0 --sched wavefront --opt wave_cta=1 > gpurun_out/r02k_cta_k$k.log 2>&1
  timeout 600 python scripts/probe.py --cfg C2 --k $k --epochs 2 --storage f16,f32 --variants 0 --sched wavefront > gpurun_out/r02k_warp_k$k.log 2>&1
  for st in f16 f32; do
    timeout 600 ncu --metrics $M --clock-control none -k regex:k_hogwild -s 3 -c 1 --csv --log-file gpurun_out/r02k_ncu_k${k}_$st.csv \
      python scripts/probe.py --cfg C2 --k $k --epochs 4 --storage $st --variants 983040 > /dev/null 2>&1
  done
done
cat gpurun_out/r02k_*.log | grep -v "^gen"
