#!/bin/bash
# run scripts/geglu_diag.py (or $SCRIPT) over the tree build and every ab/libmosaicbert_*.so, twice
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2312_17482_b200.build > /dev/null
for r in 1 2; do
  python ${SCRIPT:-scripts/geglu_diag.py}
  for f in ab/libmosaicbert_*.so; do MB_LIBRARY=$f python ${SCRIPT:-scripts/geglu_diag.py}; done
done 2>&1 | tee gpurun_out/diag.txt
