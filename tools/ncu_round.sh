#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box from the repo root):
#   1. launch list of the bench command's timed region (per-launch gpu__time_duration,
#      cold, serialised; cudaProfilerStart/Stop bracket the timed step: HP_PROFILE_RANGE=1)
#   2. ncu --set full of the root-node GEMM shapes (Gram SYRK m=8192, reconstruction 8192x4549)
#   3. ncu --set full of one root-size Jacobi round (jac_round)
# Outputs under gpurun_out/; summaries are copied into profiles/.
set -u
R=${1:-r1}
O=gpurun_out
mkdir -p $O
HP_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off -c 10000 --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/${R}_ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ --launch-skip 1 -c 1 \
  -o $O/${R}_gemm_gram8192 -f python tools/gemm_bench.py gram --m 8192 --reps 1 > $O/${R}_ncu_gram.log 2>&1
echo "gram rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ --launch-skip 1 -c 1 \
  -o $O/${R}_gemm_asm8192 -f python tools/gemm_bench.py asm --m 8192 --n 4549 --reps 1 > $O/${R}_ncu_asm.log 2>&1
echo "asm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jac_round --launch-skip 150 -c 1 \
  -o $O/${R}_jac_round -f python tools/one_node.py 30000 8192 > $O/${R}_ncu_jac.log 2>&1
echo "jac rc=$?"
