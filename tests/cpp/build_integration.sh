#!/bin/bash
# Build tests/cpp/_bin/integration_demo: the INTEGRATION.md binding (the
# document's code block, extracted verbatim) + tests/cpp/integration_main.cpp,
# against the reference's headers and sources (/root/reference/proj, present
# only in the build container).  The binary travels to the GPU box.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${REF:-/root/reference/proj}
OUT=$ROOT/tests/cpp/_bin
[ -d "$REF/include" ] || { echo "reference headers absent: not rebuilding"; exit 0; }
mkdir -p "$OUT"
python3 - "$ROOT/INTEGRATION.md" "$OUT/gpu_backend.hpp" <<'PY'
import sys
doc = open(sys.argv[1]).read()
i = doc.index("// proj/include/expmc/gpu_backend.hpp")
open(sys.argv[2], "w").write(doc[i:doc.index("```", i)])
PY
# The reference's translation units are compiled straight from where they
# lie (as oracle/Makefile does; oracle.cpp needs the absent Eigen3) into the
# test binary, with the same g++ and shared libstdc++ as libexpmc_b200.so
# (linking oracle/_ref/libexpmc_ref.so instead would put a second, static
# libstdc++ in the process).
SRCS=""
for t in sparse_matrix sampler estimator generators metrics matrix_market; do SRCS="$SRCS $REF/src/$t.cpp"; done
/usr/bin/g++ -std=c++20 -O2 -DNDEBUG -Wno-pragma-once-outside-header -I"$REF/include" -I"$ROOT/include" \
    -I"$OUT" "$ROOT/tests/cpp/integration_main.cpp" $SRCS \
    -L"$ROOT/paper_1904_12759_b200" -lexpmc_b200 \
    -Wl,-rpath,'$ORIGIN/../../../paper_1904_12759_b200' -pthread -o "$OUT/integration_demo"
echo "built $OUT/integration_demo"
