#!/bin/bash
# Round-2 time-to-Hadamard campaigns (16 seeds each), every found matrix
# re-verified on the host (H^T H = mI, balanced):
#   order 28: N = 10,000 pairs (40,000 matrices, the paper's order-28 setting),
#             F2, NC = 1, NR = 10, full restarts after 300,000 generations
#             without improvement, 240 s per seed;
#   order 36: the config-4 island (N = 312,500 pairs = 1.25M matrices), F2,
#             NC = 1, NR = 12, 120 s per seed (one attempt).
set -u
out=gpurun_out/${1:-r02tts}
mkdir -p $out
T=python\ scripts/time_to_hadamard.py
[ -z "${SKIP28:-}" ] && timeout 4200 $T --order 28 --population 10000 --fitness f2 --nc 1 --nr 10 --restart-stall 300000 \
    --seeds $(seq 0 15) --budget 240 --out $out/tts28.jsonl > /dev/null 2>> $out/err.log
[ -z "${SKIP36:-}" ] && timeout 2400 $T --order 36 --population 312500 --fitness f2 --nc 1 --nr 12 \
    --seeds $(seq 0 15) --budget 120 --out $out/tts36.jsonl > /dev/null 2>> $out/err.log
python - <<PY
import json, os
for f in ("$out/tts28.jsonl", "$out/tts36.jsonl"):
    if not os.path.exists(f): continue
    for l in open(f):
        r=json.loads(l); print(r["order"], r["seed"], r["success"], r["verified_HtH_eq_mI"], r["best_fitness"], round(r["wall_seconds"],1), r["generations"], r.get("attempts"))
PY
