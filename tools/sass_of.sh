#!/bin/bash
# SASS of the kernels of a library whose mangled name matches a pattern.
#   bash tools/sass_of.sh LIB.so PATTERN   (e.g. 'eps_unit_kernelILi2ELi1E')
LIB=$1; PAT=$2
for f in $(cuobjdump -symbols $LIB 2>/dev/null | grep -o "_Z[^ ]*$PAT[^ ]*" | sort -u); do
  cuobjdump -sass -fun $f $LIB 2>/dev/null
done
