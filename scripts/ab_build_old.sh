#!/bin/bash
# Build the committed (HEAD) library as paper_2203_03341_b200/libtcec_old.so for A/B runs.
set -e
cd "$(dirname "$0")/.."
T=$(mktemp -d)
git archive HEAD paper_2203_03341_b200/csrc include | tar -x -C "$T"
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  -I"$T/include" --expt-relaxed-constexpr -shared -o paper_2203_03341_b200/libtcec_old.so \
  "$T/paper_2203_03341_b200/csrc/tcec_capi.cu" -lcudart 2>/dev/null
rm -rf "$T"
