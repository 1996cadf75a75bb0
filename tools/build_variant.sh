#!/bin/bash
# Build libdmb200.so with extra nvcc flags into _variants/<name>/ (git-ignored, travels to the GPU box) (A/B
# tuning runs select it with DM_LIB_PATH; the product build is unaffected).
#   tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUTD=$ROOT/_variants/$NAME
mkdir -p "$OUTD"
make -C "$ROOT/paper_2601_15458_b200/csrc" -j8 OUT="$OUTD/libdmb200.so" OBJDIR="$OUTD/obj" EXTRA_NVFLAGS="$*" >/dev/null
echo "$OUTD/libdmb200.so"
