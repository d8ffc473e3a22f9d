#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box from the repo root):
#   1. launch list of the bench command (per-launch gpu__time_duration, cold, serialised)
#   2. ncu --set full of the root-node GEMM shapes (Gram SYRK m=8192, reconstruction 8192x4549)
#   3. ncu --set full of one root-size Jacobi round (jac_local / jac_apply)
# Outputs under gpurun_out/; summaries are copied into profiles/ by hand.
set -u
R=${1:-r1}
O=gpurun_out
mkdir -p $O
NCU=ncu
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/${R}_ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 1 -c 1 \
  -o $O/${R}_gemm_gram8192 -f python tools/gemm_bench.py gram --m 8192 --reps 1 > $O/${R}_ncu_gram.log 2>&1
echo "gram rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 1 -c 1 \
  -o $O/${R}_gemm_asm8192 -f python tools/gemm_bench.py asm --m 8192 --n 4549 --reps 1 > $O/${R}_ncu_asm.log 2>&1
echo "asm rc=$?"
