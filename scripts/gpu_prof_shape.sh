#!/bin/bash
# ncu --set full of the entry kernel under a forced shape.
# bash scripts/gpu_prof_shape.sh TAG CFG SHAPE [kernel-regex]
TAG=$1; CFG=$2; SH=$3; KR=${4:-entry_}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
[ "$SH" != auto ] && export EXPMC_ENTRY_SHAPE=$SH
timeout 600 python bench.py --config $CFG --kernel-only --steps 2 --warmup 1 > $OUT/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s 1 -c 1 -o $OUT/prof python bench.py --config $CFG --kernel-only --steps 2 --warmup 1 > $OUT/ncu_full.log 2>&1
tail -3 $OUT/plain.log
