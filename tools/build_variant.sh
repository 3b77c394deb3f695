#!/bin/bash
# Build a dev variant of libsconv_cuda.so from scratch (the Makefile does not
# track EXTRA, so a stale OUT dir would keep old objects):
#   tools/build_variant.sh lib_alt "-DSCONV_WS_SMALL_UNROLL=1" [git-rev]
# With a git revision the sources of that commit are built instead.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/paper_1909_09927_b200/$1
rm -rf "$OUT"
SRC=$ROOT
if [ -n "$3" ]; then
  SRC=$(mktemp -d)
  git -C "$ROOT" archive "$3" paper_1909_09927_b200/csrc include | tar -x -C "$SRC"
fi
make -s -j16 -C "$SRC/paper_1909_09927_b200/csrc" OUT="$OUT" EXTRA="$2" 2>&1 | grep -i error | head -5 || true
ls -la "$OUT/libsconv_cuda.so"
