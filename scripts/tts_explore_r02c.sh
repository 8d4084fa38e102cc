#!/bin/bash
# Round-2 order-28 campaign c: small mutation steps (per-matrix = one swap per
# child; multi NR = 2 / 4) with F2 / SQ / F1, 2 seeds x 45 s each.
set -u
out=gpurun_out/${1:-r02tts3}
mkdir -p $out
OUT=$out/tts.jsonl
T=python\ scripts/time_to_hadamard.py
for cfg in "10000 f2 per-matrix 1 1" "10000 f2 multi 1 2" "10000 f2 multi 1 4" "10000 sq per-matrix 1 1" \
           "10000 f1 per-matrix 1 1" "2500 f2 multi 1 2" "2500 f2 per-matrix 1 1" "31250 f2 per-matrix 1 1"; do
  set -- $cfg
  timeout 300 $T --order 28 --population $1 --fitness $2 --mutation $3 --nc $4 --nr $5 --seeds 200 201 --budget 45 --out $OUT > /dev/null 2>> $out/err.log
done
python - <<PY
import json
for l in open("$OUT"):
    r=json.loads(l); print(r["N"], r["fitness"], r.get("mutation"), r["nc"], r["nr"], r["seed"], r["success"], r["best_fitness"], round(r["wall_seconds"],1), r["generations"])
PY
