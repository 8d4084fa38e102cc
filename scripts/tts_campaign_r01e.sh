#!/bin/bash
# Round-1 campaign 5: small populations at order 28 (the order-20 winner's 4N = 4,000 setting,
# F2 and F1) and order 32, each run capped at 60 s.
set -u
mkdir -p gpurun_out/r01e
OUT=gpurun_out/r01e/tts.jsonl
python scripts/time_to_hadamard.py --order 28 --population 1000 --nc 2 --nr 8 --stall 200000 --seeds $(seq 0 11) --budget 60 --out $OUT
python scripts/time_to_hadamard.py --order 28 --population 1000 --nc 2 --nr 8 --fitness f1 --stall 200000 --seeds $(seq 0 5) --budget 60 --out $OUT
python scripts/time_to_hadamard.py --order 32 --population 2000 --nc 2 --nr 8 --stall 200000 --seeds $(seq 0 3) --budget 60 --out $OUT
