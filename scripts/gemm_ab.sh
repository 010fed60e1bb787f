#!/bin/bash
# GEMM timings (scripts/gemm_vs_cublas.py) of ab/libmosaicbert_prev.so vs the tree build
cd "$(dirname "$0")/.."
python -m paper_2312_17482_b200.build > /dev/null
for lib in ab/libmosaicbert_prev.so ""; do echo "== [$lib]"; MB_LIBRARY=$lib timeout 300 python scripts/gemm_vs_cublas.py; done
