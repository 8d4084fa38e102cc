#!/bin/bash
# Round-2 time-to-Hadamard exploration at order 28, config-3 island size
# (N = 31,250 pairs = 125,000 matrices): fitness (f2 / f1 / sq) x mutation
# strength x stall restarts, 2 seeds x 60 s each.  Output: gpurun_out/$1/tts.jsonl
set -u
out=gpurun_out/${1:-r02tts}
mkdir -p $out
OUT=$out/tts.jsonl
T=python\ scripts/time_to_hadamard.py
for cfg in "f2 1 10 0" "f1 1 10 0" "sq 1 10 0" "sq 1 2 0" "sq 2 4 0" "f1 1 2 0" "sq 1 4 20000" "f1 1 4 20000"; do
  set -- $cfg
  timeout 200 $T --order 28 --population 31250 --fitness $1 --nc $2 --nr $3 --stall $4 --seeds 0 1 --budget 60 --out $OUT > /dev/null 2>> $out/err.log
done
python - <<PY
import json
for l in open("$OUT"):
    r=json.loads(l); print(r["fitness"], r["nc"], r["nr"], r["stall_window"], r["seed"], r["success"], r["best_fitness"], round(r["wall_seconds"],1), r["generations"])
PY
