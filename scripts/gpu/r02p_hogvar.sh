# round 2: batch-Hogwild! shape / depth / L2-policy variants after the warp-uniform change (C2, C3)
set -x
mkdir -p gpurun_out
for c in C2 C3; do
timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f16 --variants 983040,983041,983042,983043,983072,1074724864,1343160320 > gpurun_out/r02p_f16_$c.log 2>&1
timeout 600 python scripts/probe.py --cfg $c --epochs 4 --storage f32 --variants 983040,983056,983104,983041,983042,1074724864 > gpurun_out/r02p_f32_$c.log 2>&1
done
cat gpurun_out/r02p_*.log | grep -v "^gen"
