#!/bin/bash
# round-2 tensor-core fitness kernel: parity tests + A/B sweep against the
# round-1 kernel and XOR+POPC.  Output: gpurun_out/$1/
out=gpurun_out/${1:-tc2}
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tensor_core or tc2 or fuzz" > $out/tests.log 2>&1
echo "tests_rc=$?" >> $out/tests.log
tail -n 3 $out/tests.log
for p in ${PATHS:-tc2 tc popc}; do
  timeout 600 python scripts/tc_sweep.py $1 $p > $out/sweep_$p.jsonl 2> $out/sweep_$p.err
done
[ -n "$SMALL" ] && ORDERS=20,24,28,32 VARIANTS=f2 timeout 300 python scripts/tc_sweep.py $1 popc > $out/sweep_small.jsonl 2>&1
python - <<PY
import json,glob
rows=[json.loads(l) for f in sorted(glob.glob("$out/sweep_*.jsonl")) for l in open(f) if l.startswith("{")]
for r in rows: print(r["path"], r["m"], r["variant"], "%.3g"%r["evals_per_s"], "%.3f"%r["frac_hbm"])
PY
