#!/bin/bash
# A/B of the per-call v staging (pack_v_adj variants): bash scripts/gpu_setv_ab.sh TAG variant...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
for v in "$@"; do
  if [ "$v" = default ]; then L=paper_1904_12759_b200/libexpmc_b200.so; else L=paper_1904_12759_b200/variants/lib_$v.so; fi
  echo "$v $(EXPMC_B200_LIB=$L timeout 600 python scripts/time_setv.py 2>&1 | grep set_v_device)" >> $OUT/summary.txt
done
cat $OUT/summary.txt
