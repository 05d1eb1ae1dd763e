#!/bin/bash
# Build tests/cpp/_bin/integration_demo: the INTEGRATION.md binding (the
# document's code block, extracted verbatim) + tests/cpp/integration_main.cpp,
# against the reference's headers (/root/reference/proj/include, present
# only in the build container) and the compiled reference library
# (oracle/_ref/libexpmc_ref.so).  The binary travels to the GPU box.
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
g++ -std=c++20 -O2 -Wno-pragma-once-outside-header -I"$REF/include" -I"$ROOT/include" -I"$OUT" \
    "$ROOT/tests/cpp/integration_main.cpp" \
    -L"$ROOT/oracle/_ref" -lexpmc_ref -L"$ROOT/paper_1904_12759_b200" -lexpmc_b200 \
    -Wl,-rpath,'$ORIGIN/../../../oracle/_ref:$ORIGIN/../../../paper_1904_12759_b200' -pthread \
    -o "$OUT/integration_demo"
echo "built $OUT/integration_demo"
