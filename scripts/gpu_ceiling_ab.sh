#!/bin/bash
# K3 + K6 (gather ceiling) per config for library variants: bench line fields.
# bash scripts/gpu_ceiling_ab.sh TAG "CFGS" variant...
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for c in $CFGS; do
  for v in "$@"; do
    if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
    EXPMC_B200_LIB=$L timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${v}_cfg$c.json 2> $OUT/${v}_cfg$c.err
    echo "$v cfg$c $(python -c "import json,sys; d=json.loads(open('$OUT/${v}_cfg$c.json').read().strip().splitlines()[-1]); g=d['gather_ceiling']; print(round(d['roofline']['kernel_ms'],3), 'ms K3 %.3e'%d['value'], 'K6 %.3e'%g['transitions_per_s'], 'frac %.3f'%g['frac_of_ceiling'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
