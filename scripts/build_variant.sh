#!/bin/bash
# Builds a variant of libssa with extra nvcc/g++ flags into variants/<name>/libssa.so
# usage: scripts/build_variant.sh <name> "<EXTRA flags>"
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2605_13784_b200"
make -j 16 BUILD=../variants/$name/build EXTRA="$*" libssa.so > /dev/null
mkdir -p ../variants/$name
mv libssa.so ../variants/$name/libssa.so
make -j 16 > /dev/null
