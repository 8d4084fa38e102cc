#!/bin/bash
# A/B of tc2 build variants (scripts/build_variant.sh): parity + F2 sweep each.
out=gpurun_out/${1:-tc2ab}
mkdir -p $out
for v in default ${VARIANTS_LIB}; do
  if [ $v = default ]; then unset HGA_LIB_VARIANT; else export HGA_LIB_VARIANT=$v; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tc2_many" > $out/tests_$v.log 2>&1
  echo "$v tests rc=$? $(tail -n 1 $out/tests_$v.log)"
  VARIANTS=f2 timeout 300 python scripts/tc_sweep.py $v tc2 > $out/sweep_$v.jsonl 2> $out/sweep_$v.err
  python -c "
import json
for l in open('$out/sweep_$v.jsonl'):
    r=json.loads(l); print('$v', r['m'], '%.3g'%r['evals_per_s'], '%.3f'%r['frac_hbm'])
"
done
