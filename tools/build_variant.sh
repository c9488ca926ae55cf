#!/bin/bash
# Build an experiment variant of libsaba_cuda.so with extra nvcc defines:
#   tools/build_variant.sh NAME "-DSABA_AESC_ADJ_POL=1 ..."
# -> paper_2410_14056_b200/_variants/NAME/libsaba_cuda.so; run with SABA_LIB=<that path>.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
V=$ROOT/paper_2410_14056_b200/_variants/$1
mkdir -p "$V"
make -s -C "$ROOT/paper_2410_14056_b200/csrc" OUT="$V/libsaba_cuda.so" OBJDIR="$V/_obj" EXTRA="$2"
