#!/bin/bash
# Round-1 campaign 2: F1 and stall-restart variants (results: gpurun_out/tts_r01b.jsonl)
set -u
OUT=gpurun_out/tts_r01b.jsonl
python scripts/time_to_hadamard.py --order 28 --population 10000 --nc 1 --nr 10 --fitness f1 --seeds 0 1 2 3 --budget 90 --out $OUT
python scripts/time_to_hadamard.py --order 28 --population 10000 --nc 1 --nr 10 --stall 20000 --seeds 1 2 --budget 90 --out $OUT
python scripts/time_to_hadamard.py --order 32 --population 20000 --nc 1 --nr 12 --fitness f1 --seeds 0 --budget 240 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 20000 --nc 1 --nr 12 --fitness f1 --seeds 0 --budget 300 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 50000 --nc 2 --nr 12 --fitness f1 --seeds 1 --budget 300 --out $OUT
