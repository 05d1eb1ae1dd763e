#!/bin/bash
# Accuracy legs at HEAD (entry estimator K3 on configs 1-5, Theorem-2
# estimators K4 on configs 1-4) plus the GPU test suite and smoke.
TAG=${1:-acc}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 1500 python scripts/accuracy.py > $OUT/accuracy.jsonl 2> $OUT/accuracy.err
timeout 1500 python scripts/accuracy_vector.py > $OUT/accuracy_vector.jsonl 2> $OUT/accuracy_vector.err
echo done
