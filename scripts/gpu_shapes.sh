#!/bin/bash
# K3 launch shapes (EXPMC_ENTRY_SHAPE 0: 8 blocks, 1: 7 blocks, 2: 7 blocks +
# lookahead): bit-exact model tests under each, then kernel timings.
# bash scripts/gpu_shapes.sh TAG "CFGS"
TAG=$1; CFGS=$2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for sh in 0 1 2; do
  EXPMC_ENTRY_SHAPE=$sh timeout 600 python -m pytest tests/test_gpu_parity.py -x -q \
     -k "philox_walker_matches_cpu_model or gap_edge_cases or hub_rows or sharding" > $OUT/shape${sh}_tests.log 2>&1
  echo "shape $sh tests rc=$? $(tail -1 $OUT/shape${sh}_tests.log)" >> $OUT/summary.txt
done
for c in $CFGS; do
  for sh in auto 0 1 2; do
    if [ $sh = auto ]; then unset EXPMC_ENTRY_SHAPE; else export EXPMC_ENTRY_SHAPE=$sh; fi
    timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/s${sh}_cfg$c.json 2>&1
    echo "shape=$sh cfg$c $(python -c "import json,sys; d=json.loads(open('$OUT/s${sh}_cfg$c.json').read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],3), 'ms', '%.3e'%d['value'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
unset EXPMC_ENTRY_SHAPE
cat $OUT/summary.txt
