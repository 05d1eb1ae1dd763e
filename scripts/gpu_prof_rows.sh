#!/bin/bash
# ncu --set full of K3 on the first R sampled rows of a config (long-walk configs).
# bash scripts/gpu_prof_rows.sh TAG CFG R [SHAPE]
TAG=$1; CFG=$2; R=$3; SH=${4:-auto}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
[ "$SH" != auto ] && export EXPMC_ENTRY_SHAPE=$SH
timeout 600 python scripts/k3_cfg_rows.py $CFG $R > $OUT/plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:entry_ -s 1 -c 1 -o $OUT/prof python scripts/k3_cfg_rows.py $CFG $R > $OUT/ncu_full.log 2>&1
cat $OUT/plain.log
