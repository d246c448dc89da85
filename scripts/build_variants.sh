#!/bin/bash
# Profiling experiments: build alternate copies of the library with compile-time knobs into
# paper_2312_05516_b200/variants/<name>.so (git-ignored, travels with gpurun); select one at
# run time by copying it over the product library (scripts/gpu_variants.sh).  Usage: build_variants.sh name1 "FLAGS1" name2 "FLAGS2" ...
cd "$(dirname "$0")/.."
mkdir -p paper_2312_05516_b200/variants
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  make -s -j 16 -C paper_2312_05516_b200/csrc OUT=$PWD/paper_2312_05516_b200/variants/$n.so \
       OBJDIR=$PWD/paper_2312_05516_b200/csrc/build_$n VFLAGS="$f" || exit 1
done
