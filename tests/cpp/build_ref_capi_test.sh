#!/bin/sh
# Compiles the reference's own C-ABI test suite (proj/tests/test_capi.cpp,
# unmodified, where it lies) against THIS build's include/fuseplan.h and
# libfuseplan_b200.so, with a doctest shim; output oracle/_ref/ref_test_capi.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${FUSEPLAN_REFERENCE:-/root/reference}/proj/tests/test_capi.cpp
mkdir -p "$ROOT/oracle/_ref"
g++ -std=c++20 -O1 -DSHIM_MAIN \
  -DFUSEPLAN_DATA_DIR="\"$ROOT/paper_1509_04394_b200/data\"" \
  -I"$ROOT/tests/cpp/doctest_shim" -I"$ROOT/include" \
  "$REF" -o "$ROOT/oracle/_ref/ref_test_capi" \
  -L"$ROOT/paper_1509_04394_b200" -lfuseplan_b200 \
  -Wl,-rpath,"$ROOT/paper_1509_04394_b200"
echo "$ROOT/oracle/_ref/ref_test_capi"
