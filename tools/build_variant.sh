#!/bin/bash
# Build the product library of a commit (or of the working tree: WT) into
# variants/NAME/libbnmc_b200.so for same-box A/B runs (BNMC_B200_LIB=...).
# Extra nvcc flags (e.g. -DBNMC_KEEP_Y=0) come from $NVEXTRA.
#   [NVEXTRA=...] bash tools/build_variant.sh NAME COMMIT|WT
set -eu
NAME=$1; REV=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/tmp/bnmc_wt_$NAME
mkdir -p "$ROOT/variants/$NAME"
rm -rf "$SRC"; git -C "$ROOT" worktree prune
if [ "$REV" = WT ]; then
  mkdir -p "$SRC"; cp -r "$ROOT/include" "$SRC/"; mkdir -p "$SRC/paper_1210_5128_b200"
  cp -r "$ROOT/paper_1210_5128_b200/csrc" "$SRC/paper_1210_5128_b200/"; rm -rf "$SRC/paper_1210_5128_b200/csrc/_build"
else
  git -C "$ROOT" worktree add -f --detach "$SRC" "$REV" >/dev/null
fi
make -s -j8 -C "$SRC/paper_1210_5128_b200/csrc" NVEXTRA="${NVEXTRA:-}" \
  "$SRC/paper_1210_5128_b200/csrc/../libbnmc_b200.so" 2>&1 | grep -v "spill" || true
cp "$SRC/paper_1210_5128_b200/libbnmc_b200.so" "$ROOT/variants/$NAME/libbnmc_b200.so"
if [ "$REV" = WT ]; then rm -rf "$SRC"; else git -C "$ROOT" worktree remove --force "$SRC"; fi
echo "variants/$NAME/libbnmc_b200.so <- $REV ${NVEXTRA:-}"
