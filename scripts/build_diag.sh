#!/bin/bash
# Diagnostic builds of the working tree with extra nvcc defines into ab/libmosaicbert_<name>.so:
#   scripts/build_diag.sh <name> "-DMB_DIAG_X=1 ..."
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
MB_EXTRA_FLAGS="$2" MB_OBJ_SUFFIX="_$1" MB_LIB_OUT="ab/libmosaicbert_$1.so" python -m paper_2312_17482_b200.build > /dev/null
echo "ab/libmosaicbert_$1.so <- working tree + $2"
