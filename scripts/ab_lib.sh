#!/bin/bash
# Local helper: build the committed HEAD version of the library as build_ab/libmoeshard_base.so
# next to the working-tree build, so a GPU call can A/B the two binaries on one box:
#   scripts/ab_lib.sh            (here)  then on the box:
#   bash scripts/ab_env.sh MOESHARD_LIB_PATH=$PWD/build_ab/libmoeshard_base.so X=1 ...
set -e
cd /root/repo
rm -rf /tmp/ab_src && mkdir -p /tmp/ab_src build_ab
git archive HEAD paper_2503_08467_b200 include | tar -x -C /tmp/ab_src
python - <<'PY'
import sys, importlib.util
spec = importlib.util.spec_from_file_location("b", "/tmp/ab_src/paper_2503_08467_b200/_build.py")
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
print(m.build(force=True))
PY
cp /tmp/ab_src/paper_2503_08467_b200/libmoeshard.so build_ab/libmoeshard_base.so
python paper_2503_08467_b200/_build.py > /dev/null
ls -la build_ab
