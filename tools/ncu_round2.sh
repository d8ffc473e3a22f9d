#!/usr/bin/env bash
# Round-2 profiling pass after the tridiagonal eigensolver (run on the GPU box from the repo root):
#   1. launch list of the bench command's timed step (per-launch gpu__time_duration; cold, serialised)
#   2. ncu --set full of the first (largest, HBM-bound) sytrd_panel launch of a config-1-root-sized solve
#   3. ncu --set full of a mid-solve sytrd_panel launch (L2-resident trailing matrix)
set -u
R=${1:-r2h}
O=gpurun_out
mkdir -p $O
HP_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off -c 12000 --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/${R}_ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sytrd_panel -c 1 \
  -o $O/${R}_sytrd_panel_first -f python tools/tri_study.py 30000 8192 1 0 tri > $O/${R}_ncu_sytrd1.log 2>&1
echo "sytrd first rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sytrd_panel --launch-skip 55 -c 1 \
  -o $O/${R}_sytrd_panel_mid -f python tools/tri_study.py 30000 8192 1 0 tri > $O/${R}_ncu_sytrd2.log 2>&1
echo "sytrd mid rc=$?"
