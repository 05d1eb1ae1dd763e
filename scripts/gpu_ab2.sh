#!/bin/bash
# A/B of library variants: bit-exact K3 model tests, then kernel-only timing.
# bash scripts/gpu_ab2.sh TAG "CFGS" variant...   ("default" = the in-tree build)
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for v in "$@"; do
  if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
  EXPMC_B200_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -x -q \
     -k "philox_walker_matches_cpu_model or gap_edge_cases or hub_rows" > $OUT/${v}_tests.log 2>&1
  echo "$v tests rc=$? $(tail -1 $OUT/${v}_tests.log)" >> $OUT/summary.txt
done
for c in $CFGS; do
  for v in "$@"; do
    if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
    EXPMC_B200_LIB=$L timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/${v}_cfg$c.json 2>&1
    echo "$v cfg$c $(python -c "import json,sys; d=json.loads(open('$OUT/${v}_cfg$c.json').read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],3), 'ms', '%.3e'%d['value'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
