#!/bin/bash
# Wide randomised bit-exact sweep of the entry walker (default and self-checking
# builds) and the torchrun-launched bench lines: bash scripts/gpu_soak_round.sh TAG
TAG=${1:-soak}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
EXPMC_SOAK_CASES=2000 timeout 1200 python -m pytest tests/test_gpu_soak.py -x -q > $OUT/soak_default.log 2>&1; echo "rc=$?" >> $OUT/soak_default.log
[ -f paper_1904_12759_b200/variants/lib_checks.so ] && { EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_checks.so EXPMC_SOAK_CASES=600 timeout 1200 python -m pytest tests/test_gpu_soak.py -x -q > $OUT/soak_checks.log 2>&1; echo "rc=$?" >> $OUT/soak_checks.log; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 > $OUT/torchrun_bench_cfg5.json 2> $OUT/torchrun_bench_cfg5.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > $OUT/torchrun_ref_cfg5.json 2> $OUT/torchrun_ref_cfg5.err
tail -n 2 $OUT/soak_default.log; tail -n 2 $OUT/soak_checks.log; cut -c1-200 $OUT/torchrun_bench_cfg5.json; cut -c1-200 $OUT/torchrun_ref_cfg5.json
