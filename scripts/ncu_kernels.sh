#!/bin/bash
# Full ncu captures of the int8 tcgen05 GEMM (c5 sketch shape, c2 E3 shape) and the fp32 pair
# quantiser (c2 bench) for the round's profile summaries.
O=${1:-gpurun_out/r01}
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:igemm_tn_kernel -s 3 -c 1 \
  -o $O/ncu_igemm_c5sketch python scripts/igemm_once.py 131072 1056 8192 f64 > $O/ncu_igemm1.log 2>&1
echo "igemm c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:igemm_tn_kernel -s 3 -c 1 \
  -o $O/ncu_igemm_c2e3 python scripts/igemm_once.py 4096 4096 256 f32 > $O/ncu_igemm2.log 2>&1
echo "igemm c2 E3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_tile_kernel -c 1 \
  -o $O/ncu_quant_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_quant.log 2>&1
echo "quant rc=$?"
