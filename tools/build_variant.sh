#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh <name> "<-D flags>"
# -> variants/<name>.so (time with SDR_LIB_PATH=variants/<name>.so python tools/time_ab.py)
set -e
cd "$(dirname "$0")/../paper_2509_07003_b200/csrc"
mkdir -p ../../variants
make -s OBJDIR=../_objv_$1 LIB=../../variants/$1.so \
  NVFLAGS="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $2" -j4
rm -rf ../_objv_$1  # objects are 17 MB per variant; only the .so travels
