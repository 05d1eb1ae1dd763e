#!/bin/bash
# A/B of library variants at given (config:shape) points, kernel-only timing.
# bash scripts/gpu_ab3.sh TAG "5:0 4:1 ..." variant...   ("default" = the in-tree build)
TAG=$1; PTS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for pt in $PTS; do
  c=${pt%%:*}; sh=${pt#*:}
  for v in "$@"; do
    if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
    if [ $sh = auto ]; then unset EXPMC_ENTRY_SHAPE; else export EXPMC_ENTRY_SHAPE=$sh; fi
    EXPMC_B200_LIB=$L timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/${v}_cfg${c}_s$sh.json 2> $OUT/${v}_cfg${c}_s$sh.err
    echo "$v cfg$c shape=$sh $(python -c "import json,sys; d=json.loads(open('$OUT/${v}_cfg${c}_s$sh.json').read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],3), 'ms', '%.3e'%d['value'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
