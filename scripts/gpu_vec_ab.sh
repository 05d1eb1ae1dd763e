#!/bin/bash
# Theorem-2 estimators (K4) for library variants: ms per host call.
# bash scripts/gpu_vec_ab.sh TAG "CFGS" variant...
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for v in "$@"; do
  if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
  EXPMC_B200_LIB=$L timeout 1500 python scripts/bench_vector.py --configs $CFGS --steps 3 --no-cpu > $OUT/$v.jsonl 2> $OUT/$v.err
  python - "$OUT/$v.jsonl" "$v" >> $OUT/summary.txt <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[2], d['estimator'], d['config'], round(d['gpu']['ms_per_call'],3),'ms', '%.3e'%d['gpu']['transitions_per_s'])
PY
done
cat $OUT/summary.txt
