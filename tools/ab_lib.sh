#!/bin/bash
# A/B of library variants on cfg5 (or $CFG): bench K2 ms + ms/step, alternating.
# Usage: tools/ab_lib.sh OUTDIR lib1 lib2 ...   ("main" = the in-tree build)
out=$1; shift
mkdir -p $out
CFG=${CFG:-5}
for rep in 1 2; do
  for lib in "$@"; do
    tag=$(basename $lib .so)
    if [ "$lib" = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
    timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $out/b_${tag}_$rep.json 2> $out/b_${tag}_$rep.err
    python - $out/b_${tag}_$rep.json $tag $rep <<'PY' >> $out/summary.txt
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
r = d["roofline"]
print(sys.argv[2], sys.argv[3], "ms/step %.4f K2 %.4f frac %.3f MHz %s %s" % (d["ms_per_step"], r["kernel_ms"], r["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
PY
  done
done
unset CORR2D_LIB
cat $out/summary.txt
