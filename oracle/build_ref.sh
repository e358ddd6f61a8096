#!/usr/bin/env bash
# Build the reference's own hot-path headers IN PLACE into oracle/_ref/libhelmref.so.
# TEST INFRASTRUCTURE (oracle pin + CPU reference arm).  Nothing is copied from
# /root/reference: the headers are compiled where they lie via -I.  Third-party
# pieces the reference expects but this image lacks are replaced as follows:
#   Eigen         -> oracle/ref/shim/Eigen (from-scratch API subset; GEMM = OpenBLAS sgemm,
#                    single-threaded, standing in for Eigen's GEMM)
#   nlohmann/json -> the copy vendored under cudnn_frontend/thirdparty (datagen.hpp include)
# Flags follow proj/CMakeLists.txt:11 (-O3, C++20); -march=x86-64-v3 instead of
# -march=native so the prebuilt .so also runs on the GPU box host CPU.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF_INC="${HELM_REF_INCLUDE:-/root/reference/proj/include}"
if [ ! -d "$REF_INC/helmbench" ]; then
  echo "reference headers not found at $REF_INC (skipping oracle/_ref build)" >&2
  exit 3
fi
PY=${PYTHON:-python}
SITE="$($PY -c 'import sysconfig;print(sysconfig.get_paths()["purelib"])')"
JSON_INC="$SITE/include/cudnn_frontend/thirdparty"
BLAS_DIR="$SITE/opencv_python_headless.libs"
BLAS_LIB="$(ls "$BLAS_DIR"/libopenblas*.so 2>/dev/null | head -1)"
if [ -z "$BLAS_LIB" ]; then echo "OpenBLAS not found under $BLAS_DIR" >&2; exit 4; fi
mkdir -p "$HERE/_ref"
g++ -std=c++20 -O3 -march=x86-64-v3 -mtune=native -fPIC -shared \
  -I"$HERE/ref/shim" -I"$REF_INC" -I"$JSON_INC" \
  -o "$HERE/_ref/libhelmref.so" "$HERE/ref/ref_capi.cpp" \
  "$BLAS_LIB" -Wl,--disable-new-dtags,-rpath,"$BLAS_DIR" -Wl,--allow-shlib-undefined -pthread
echo "built $HERE/_ref/libhelmref.so"
