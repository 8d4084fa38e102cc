#!/bin/bash
# Round-1 time-to-Hadamard campaign on one B200 (results: gpurun_out/tts_r01.jsonl)
set -u
OUT=gpurun_out/tts_r01.jsonl
# order 20, paper section 4.4 setting (N=1000, NC=2, NR=8), F2 and F1 with stall restart
python scripts/time_to_hadamard.py --order 20 --population 1000 --nc 2 --nr 8 --seeds 2 3 4 5 --budget 60 --out $OUT
python scripts/time_to_hadamard.py --order 20 --population 10000 --nc 4 --nr 2 --seeds 0 1 --budget 60 --out $OUT
# order 28: paper setting (N=10^4, NC=1, NR=10) and the config-3 island size (N=31,250 = 125k matrices)
python scripts/time_to_hadamard.py --order 28 --population 10000 --nc 1 --nr 10 --seeds 0 1 2 --budget 120 --out $OUT
python scripts/time_to_hadamard.py --order 28 --population 31250 --nc 1 --nr 10 --seeds 0 1 --budget 120 --out $OUT
# order 32 (paper: N=2*10^4, NC=1, NR=12) and order 36 exploratory
python scripts/time_to_hadamard.py --order 32 --population 20000 --nc 1 --nr 12 --seeds 0 --budget 180 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 20000 --nc 1 --nr 12 --seeds 0 --budget 240 --stall 2000 --out $OUT
python scripts/time_to_hadamard.py --order 36 --population 312500 --nc 1 --nr 12 --seeds 0 --budget 240 --out $OUT
