#!/bin/bash
# Build a copy of the working tree with extra nvcc defines into tmp_variants/<name> (git-ignored,
# travels to the GPU box) for A/B timing:  tools/variant.sh <name> [-DFOO=1 ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1
shift
dst=$ROOT/tmp_variants/$name
rm -rf "$dst"
mkdir -p "$dst"
(cd "$ROOT" && tar cf - --exclude=.git --exclude=tmp_variants --exclude=gpurun_out --exclude='*.so' . ) | tar xf - -C "$dst"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  "$@" -o "$dst/paper_1901_00913_b200/libkb_b200.so" "$dst/paper_1901_00913_b200/csrc/kb_capi.cu"
echo "built $dst $*"
