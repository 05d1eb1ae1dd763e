#!/bin/bash
OUT=gpurun_out/r2b; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1
echo "tests rc=$? $(tail -1 $OUT/gpu_tests.log)" >> $OUT/summary.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err
echo "ref rc=$?" >> $OUT/summary.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/summary.txt
python scripts/time_single_entry.py > $OUT/single_entry.json 2> $OUT/single_entry.err
echo "single rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
