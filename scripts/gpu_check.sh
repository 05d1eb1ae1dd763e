#!/bin/bash
# smoke + GPU tests + default bench line (cfg 5) + extra kernel-only configs
TAG=${1:-check}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in "$@"; do
  timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 3 > $OUT/k_cfg$c.json 2>&1
done
echo done
