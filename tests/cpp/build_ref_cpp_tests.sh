#!/bin/sh
# Compiles the reference's own C++ test suites for the planner, tiling and
# dependency layers (proj/tests/test_planner.cpp, test_tiling.cpp,
# test_dependency.cpp -- unmodified, where they lie, with their helpers.hpp)
# against THIS build's public C++ headers (include/fuseplan/*.hpp) and
# libfuseplan_b200.so, with the doctest shim; output oracle/_ref/ref_test_cpp.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${FUSEPLAN_REFERENCE:-/root/reference}/proj/tests
JSON_DIR=${FUSEPLAN_JSON_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
mkdir -p "$ROOT/oracle/_ref"
printf '#define SHIM_MAIN\n#include "doctest.h"\n' > "$ROOT/oracle/_ref/shim_main.cpp"
g++ -std=c++20 -O1 -ffp-contract=off \
  -DFUSEPLAN_DATA_DIR="\"$ROOT/paper_1509_04394_b200/data\"" \
  -DFUSEPLAN_GOLDEN_DIR="\"$REF/golden\"" \
  -I"$ROOT/tests/cpp/doctest_shim" -I"$ROOT/include" -I"$REF" -I"$JSON_DIR" \
  "$ROOT/oracle/_ref/shim_main.cpp" "$REF/test_planner.cpp" "$REF/test_tiling.cpp" \
  "$REF/test_dependency.cpp" -o "$ROOT/oracle/_ref/ref_test_cpp" \
  -L"$ROOT/paper_1509_04394_b200" -lfuseplan_b200 \
  -Wl,-rpath,"$ROOT/paper_1509_04394_b200"
echo "$ROOT/oracle/_ref/ref_test_cpp"
