#!/bin/bash
# Round-2 order-28 campaign b: success probability per 30 s attempt at the
# paper's population (N = 10,000 = 40,000 matrices) and the config-3 island
# (N = 31,250), F2, NC = 1, NR in {10, 6}; 8 seeds each.
set -u
out=gpurun_out/${1:-r02tts2}
mkdir -p $out
OUT=$out/tts.jsonl
T=python\ scripts/time_to_hadamard.py
for cfg in "10000 1 10" "10000 1 6" "31250 1 6" "10000 2 8"; do
  set -- $cfg
  timeout 400 $T --order 28 --population $1 --fitness f2 --nc $2 --nr $3 --seeds 100 101 102 103 104 105 106 107 --budget 30 --out $OUT > /dev/null 2>> $out/err.log
done
python - <<PY
import json
for l in open("$OUT"):
    r=json.loads(l); print(r["N"], r["nc"], r["nr"], r["seed"], r["success"], r["best_fitness"], round(r["wall_seconds"],1), r["generations"])
PY
