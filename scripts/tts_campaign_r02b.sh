#!/bin/bash
# Round-2 time-to-Hadamard campaign, second half: order 36 at the config-4
# island size (seeds 9-15 of the 16-seed set; 0-8 ran in r02tts4), then order
# 28 with full restarts after 150,000 stalled generations, 300 s per seed
# (SEEDS28 env: which seeds).
set -u
out=gpurun_out/${1:-r02tts5}
mkdir -p $out
T=python\ scripts/time_to_hadamard.py
[ -n "${SEEDS36:-}" ] && timeout 1500 $T --order 36 --population 312500 --fitness f2 --nc 1 --nr 12 \
    --seeds $SEEDS36 --budget 120 --out $out/tts36.jsonl > /dev/null 2>> $out/err.log
[ -n "${SEEDS28:-}" ] && timeout 3300 $T --order 28 --population 10000 --fitness f2 --nc 1 --nr 10 --restart-stall 150000 \
    --seeds $SEEDS28 --budget 300 --out $out/tts28.jsonl > /dev/null 2>> $out/err.log
exit 0
