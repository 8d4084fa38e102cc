#!/bin/bash
# role ablation of the tc2 kernel (HGA_TC_FLAGS): which role sets the pace
out=gpurun_out/${1:-tc2roles}
mkdir -p $out
for f in 0 2 4 8 6 10 12 14; do
  HGA_TC_FLAGS=$f ORDERS=48,64 VARIANTS=f2 timeout 300 python scripts/tc_sweep.py f$f tc2 > $out/roles_$f.jsonl 2>&1
  python -c "
import json
for l in open('$out/roles_$f.jsonl'):
    if l.startswith('{'): r=json.loads(l); print('flags $f', r['m'], '%.3g'%r['evals_per_s'], '%.3f'%r['frac_hbm'])
"
done
