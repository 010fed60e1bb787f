#!/bin/bash
# Build the library of git revision $1 (default HEAD) into ab/libmosaicbert_<name>.so for A/B runs:
#   MB_LIBRARY=ab/libmosaicbert_<name>.so python bench.py ...
set -e
cd "$(dirname "$0")/.."
rev=${1:-HEAD}; name=${2:-base}
tmp=$(mktemp -d /tmp/ab.XXXXXX)
git archive "$rev" | tar -x -C "$tmp"
(cd "$tmp" && python -m paper_2312_17482_b200.build > /dev/null)
mkdir -p ab
cp "$tmp/paper_2312_17482_b200/libmosaicbert.so" "ab/libmosaicbert_$name.so"
rm -rf "$tmp"
echo "ab/libmosaicbert_$name.so <- $rev"
