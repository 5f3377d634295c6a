#!/bin/bash
# Build an experiment variant of libpss.so: tools/variant.sh OUT.so -DFLAG ...
# (timing experiments only; load with PSS_LIB=OUT.so)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
  -I "$ROOT/include" "$@" -o "$OUT" "$ROOT"/paper_1606_04669_b200/csrc/*.cu
