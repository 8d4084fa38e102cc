#!/bin/bash
# Round-1 campaign 3: long runs at orders 32 and 36 (results: gpurun_out/tts_r01c.jsonl)
set -u
OUT=gpurun_out/tts_r01c.jsonl
python scripts/time_to_hadamard.py --order 32 --population 20000 --nc 1 --nr 12 --seeds 1 --budget 1200 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 20000 --nc 1 --nr 12 --seeds 2 --budget 1200 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 312500 --nc 1 --nr 12 --seeds 3 --budget 900 --out $OUT
