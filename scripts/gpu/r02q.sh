# round 2: new batch-Hogwild! defaults (fp16 k=128: 32 lanes x 8 B; fp32 k=128: one rating per group),
# parity, throughput, the shuffled Hugewiki load footprint, CTA vs warp wavefront on the Hugewiki shape
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -q -p no:cacheprovider -x > gpurun_out/r02q_pytest.log 2>&1
tail -3 gpurun_out/r02q_pytest.log
for c in C2 C3 C4-rows10; do
  timeout 600 python scripts/probe.py --cfg $c --epochs 5 --storage f16,f32 --variants -1 > gpurun_out/r02q_hog_$c.log 2>&1
done
cat gpurun_out/r02q_hog_*.log
timeout 900 python scripts/c4_shuffled_load.py > gpurun_out/r02q_c4_shuffled_load.json 2> gpurun_out/r02q_c4_shuffled_load.err
cat gpurun_out/r02q_c4_shuffled_load.json; tail -3 gpurun_out/r02q_c4_shuffled_load.err
timeout 1800 python scripts/trace_compare.py --cfg C4 --storage f16 --epochs 4 --shuffle 0 \
  --scheds wavefront,wavefront_cta,wavefront_cta@variant=134217728 > gpurun_out/r02q_c4_wavefront.jsonl 2> gpurun_out/r02q_c4_wavefront.err
cat gpurun_out/r02q_c4_wavefront.jsonl
