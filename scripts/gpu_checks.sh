#!/bin/bash
# The self-checking K3 build (-DEXPMC_CHECKS: device-side asserts on the
# ticket ring, task ring, gather bounds and accumulation order) under the
# bit-exact model tests, every launch shape, row sharding, and full-size
# slices of configs 2, 4 and 5.  compute-sanitizer is closed on this pool.
# bash scripts/gpu_checks.sh TAG
TAG=${1:-checks}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
export EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_checks.so
for sh in 0 1; do
  EXPMC_ENTRY_SHAPE=$sh timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q \
     -k "philox_walker_matches_cpu_model or gap_edge_cases or hub_rows or sharding or weighted or kat or device_api" > $OUT/shape${sh}_tests.log 2>&1
  echo "checks build, shape $sh: rc=$? $(tail -1 $OUT/shape${sh}_tests.log)" | tee -a $OUT/summary.txt
done
unset EXPMC_ENTRY_SHAPE
for c in "2 100000" "4 4096" "5 200000" "1 4096"; do
  set -- $c
  timeout 1200 python scripts/k3_cfg_rows.py $1 $2 > $OUT/cfg$1.log 2>&1
  echo "checks build, config $1 first $2 rows: rc=$? $(tail -1 $OUT/cfg$1.log)" | tee -a $OUT/summary.txt
done
grep -l "check failed" $OUT/*.log && echo "CHECK FAILURES" | tee -a $OUT/summary.txt || echo "no device check fired" | tee -a $OUT/summary.txt
