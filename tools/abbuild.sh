#!/bin/bash
# Build libhelmgpu.so from a git revision (default HEAD) into build/ab/<rev>/ for
# A/B timing on the GPU box: HB_LIB_PATH=build/ab/<rev>/libhelmgpu.so python ...
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2203_11025_b200 include | tar -x -C "$tmp"
python "$tmp/paper_2203_11025_b200/build.py" > /dev/null 2>&1
mkdir -p "$root/build/ab/$rev"
cp "$tmp/paper_2203_11025_b200/libhelmgpu.so" "$root/build/ab/$rev/libhelmgpu.so"
rm -rf "$tmp"
echo "$root/build/ab/$rev/libhelmgpu.so"
