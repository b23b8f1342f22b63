#!/bin/bash
# Experiment build (here, no GPU): compile libmoeshard.so with extra nvcc defines into
# build_ab/<name>/libmoeshard.so, for a same-box A/B with scripts/ab_variants.sh.
#   bash scripts/build_variant.sh <name> [-DFOO=1 ...]
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build_ab/$NAME
mkdir -p $OUT/obj
NCCL_INC=$(python -c "import nvidia.nccl as n, os; print(os.path.join(list(n.__path__)[0], 'include'))")
for f in $ROOT/paper_2503_08467_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a \
    -Xcompiler -fPIC -I $ROOT/include -I $NCCL_INC "$@" -c $f -o $OUT/obj/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT/libmoeshard.so $OUT/obj/*.o -ldl
rm -rf $OUT/obj
echo $OUT/libmoeshard.so
