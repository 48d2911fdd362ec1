#!/bin/bash
# Build the library with extra nvcc defines into variants/NAME.so (for tools/ab.sh).
#   bash tools/build_variant.sh NAME "-DDS_MINB_SMALL=5 ..."
set -e
NAME=$1; shift
mkdir -p variants build/variant_$NAME
make -s -C paper_1506_02226_b200/csrc OUT=../../variants/$NAME.so OBJDIR=../../build/variant_$NAME EXTRA="$*" 2>&1 | grep -v "^$" | grep -iv "spill" || true
ls -la variants/$NAME.so
