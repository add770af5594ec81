#!/bin/bash
# Builds the -DSSA_GTRACE variant of libssa into variants/gtrace/libssa.so (the
# in-tree libssa.so is rebuilt normally afterwards).
set -e
cd "$(dirname "$0")/../paper_2605_13784_b200"
make -j 16 BUILD=../variants/gtrace/build EXTRA=-DSSA_GTRACE libssa.so > /dev/null
mkdir -p ../variants/gtrace
mv libssa.so ../variants/gtrace/libssa.so
make -j 16 > /dev/null
