#!/bin/bash
# K3S (phase-scheduled short-walk kernel) against entry_walk_kernel: the
# bit-exact CPU-model tests under each forced shape (EXPMC_ENTRY_SHAPE 0: 8
# blocks, 1: 7 blocks, 3: K3S), then kernel timings per config.
# bash scripts/gpu_k3s.sh TAG "CFGS" ["SHAPES"]
TAG=$1; CFGS=$2; SHAPES=${3:-"auto 0 3"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for sh in ${TEST_SHAPES:-3 0 1}; do
  EXPMC_ENTRY_SHAPE=$sh timeout 900 python -m pytest tests/test_gpu_parity.py -x -q \
     -k "philox_walker_matches_cpu_model or gap_edge_cases or hub_rows or sharding or weighted" > $OUT/shape${sh}_tests.log 2>&1
  echo "shape $sh tests rc=$? $(tail -1 $OUT/shape${sh}_tests.log)" >> $OUT/summary.txt
done
for c in $CFGS; do
  for sh in $SHAPES; do
    if [ $sh = auto ]; then unset EXPMC_ENTRY_SHAPE; else export EXPMC_ENTRY_SHAPE=$sh; fi
    EXPMC_DEBUG=1 timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/s${sh}_cfg$c.json 2> $OUT/s${sh}_cfg$c.err
    echo "shape=$sh cfg$c $(python -c "import json,sys; d=json.loads(open('$OUT/s${sh}_cfg$c.json').read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],3), 'ms', '%.3e'%d['value'])" 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
unset EXPMC_ENTRY_SHAPE
cat $OUT/summary.txt
