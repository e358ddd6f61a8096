#!/usr/bin/env bash
# Build tests/cpp/_build/dropin against the reference headers (in place) + libhelmgpu.
# TEST INFRASTRUCTURE; needs /root/reference (here), the binary travels to the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$(dirname "$HERE")")"
REF_INC="${HELM_REF_INCLUDE:-/root/reference/proj/include}"
[ -d "$REF_INC/helmbench" ] || { echo "no reference headers; skip" >&2; exit 3; }
PY=${PYTHON:-python}
SITE="$($PY -c 'import sysconfig;print(sysconfig.get_paths()["purelib"])')"
BLAS_DIR="$SITE/opencv_python_headless.libs"
BLAS_LIB="$(ls "$BLAS_DIR"/libopenblas*.so | head -1)"
mkdir -p "$HERE/_build"
g++ -std=c++20 -O2 -I"$ROOT/oracle/ref/shim" -I"$REF_INC" -I"$ROOT/include" \
  -o "$HERE/_build/dropin" "$HERE/dropin.cpp" \
  -L"$ROOT/paper_2203_11025_b200" -l:libhelmgpu.so -Wl,--disable-new-dtags,-rpath,'$ORIGIN/../../../paper_2203_11025_b200' \
  "$BLAS_LIB" -Wl,-rpath,"$BLAS_DIR" -Wl,--allow-shlib-undefined -pthread
echo "built $HERE/_build/dropin"
