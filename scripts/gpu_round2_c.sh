#!/bin/bash
OUT=gpurun_out/r2c; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > $OUT/gpu_tests.log 2>&1
echo "tests rc=$? $(tail -1 $OUT/gpu_tests.log)" >> $OUT/summary.txt
python scripts/time_single_entry.py > $OUT/single_entry.json 2> $OUT/single_entry.err
echo "single rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
