#!/usr/bin/env bash
# Final round-2 profiling pass (run on the GPU box from the repo root, after the same commands exited 0
# without ncu):
#   1. launch list of the bench command's timed step (per-launch gpu__time_duration; cold, serialised)
#   2. ncu --set full of the config-1 root Gramian (8,192 columns x 200,000 rows: first gemm_tma_kernel launch)
#   3. ncu --set full of a leaf Gramian (512 columns: split-K launch whose diagonal tiles take mma_ktile_diag)
set -u
R=${1:-r2n}
O=gpurun_out
mkdir -p $O
HP_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off -c 12000 --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/${R}_ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -c 1 \
  -o $O/${R}_gemm_gram8192 -f python tools/one_node.py 200000 8192 > $O/${R}_ncu_gram8192.log 2>&1
echo "root gram rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -c 1 \
  -o $O/${R}_gemm_gram512 -f python tools/one_node.py 200000 512 > $O/${R}_ncu_gram512.log 2>&1
echo "leaf gram rc=$?"
