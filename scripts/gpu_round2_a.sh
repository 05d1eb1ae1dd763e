#!/bin/bash
# GPU tests + kernel timing with the resident-block choice forced both ways.
OUT=gpurun_out/r2a; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1
echo "tests rc=$? $(tail -1 $OUT/gpu_tests.log)" >> $OUT/summary.txt
for c in 5 1 2 3 4; do
  for b in auto 7 8; do
    if [ $b = auto ]; then unset EXPMC_ENTRY_BLOCKS; else export EXPMC_ENTRY_BLOCKS=$b; fi
    timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/b${b}_cfg$c.json 2>&1
    echo "blocks=$b cfg$c $(python -c "import json,sys; d=json.loads(open('$OUT/b${b}_cfg$c.json').read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],3), 'ms', '%.3e'%d['value'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
unset EXPMC_ENTRY_BLOCKS
cat $OUT/summary.txt
