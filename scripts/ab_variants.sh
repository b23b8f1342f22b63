#!/bin/bash
# Same-box A/B of prebuilt library variants (run under gpurun): for each repetition and
# each variant in build_ab/, put its libmoeshard.so in place and run the probe command.
#   bash scripts/ab_variants.sh "<probe command>" <reps> <variant> [<variant> ...]
CMD=$1; REPS=$2; shift 2
LIB=paper_2503_08467_b200/libmoeshard.so
cp $LIB /tmp/ab_lib_orig
mkdir -p gpurun_out
for rep in $(seq $REPS); do
  for v in "$@"; do
    cp build_ab/$v/libmoeshard.so $LIB
    echo "$v $rep $(timeout 600 $CMD 2>/dev/null | tail -1)"
  done
done | tee gpurun_out/ab_variants.txt
cp /tmp/ab_lib_orig $LIB
