#!/bin/bash
# Build an alternate libfc2.so under variants/<name>/ with extra nvcc defines (dev tool).
#   tools/build_variant.sh <name> "-DFOO=1 -DBAR=0"
set -e
name=$1; shift
make -s -j"$(nproc)" OBJ=variants/$name/_build LIB=variants/$name/libfc2.so EXTRA="$*" all > /dev/null
echo "built variants/$name/libfc2.so ($*)"
