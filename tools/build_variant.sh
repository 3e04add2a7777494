#!/bin/bash
# Build libwfpg_b200.so of another git revision (A/B measurements on one box):
#   tools/build_variant.sh <rev> <out.so>     then   WFPG_LIB=<out.so> python bench.py ...
set -e
REV=$1; OUT=$(realpath -m "$2")
REPO=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$REPO" worktree add -q --detach "$TMP" "$REV"
make -s -C "$TMP/paper_2405_06997_b200/csrc" -j8 OUT="$OUT" 2>&1 | grep -v "spill\|^$" || true
git -C "$REPO" worktree remove --force "$TMP"
ls -la "$OUT"
