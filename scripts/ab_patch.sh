#!/bin/bash
# Same-box A/B of a source patch (run under gpurun; the box's copy of the repo is scratch):
#   bash scripts/ab_patch.sh <tag> <file> <python-literal old> <python-literal new> [bench args]
# builds and benches A (as committed) and B (patched), twice each, interleaved A B A B.
TAG=$1; FILE=$2; OLD=$3; NEW=$4; shift 4
ARGS=${@:-"--steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0"}
cp $FILE /tmp/ab_orig
python - "$FILE" "$OLD" "$NEW" <<'PY'
import sys, ast
f, old, new = sys.argv[1], ast.literal_eval(sys.argv[2]), ast.literal_eval(sys.argv[3])
s = open(f).read(); assert old in s, "patch anchor not found"; open("/tmp/ab_patched", "w").write(s.replace(old, new))
PY
for rep in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp /tmp/ab_orig $FILE; else cp /tmp/ab_patched $FILE; fi
    python paper_2503_08467_b200/_build.py > /dev/null || exit 1
    python bench.py $ARGS > gpurun_out/ab_${TAG}_${v}${rep}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_${v}${rep}.json'));print('$v$rep', round(d['ms_per_step']*1e3,2), 'us', {k:v['us'] for k,v in d['kernels_us'].items()})"
  done
done
cp /tmp/ab_orig $FILE
