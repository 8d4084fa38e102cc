#!/bin/bash
# Round-2 order-28 campaign (final protocol): N = 10,000 pairs (40,000
# matrices, the paper's order-28 setting), F2, NC = 1, NR = 10, full restarts
# after 300,000 generations without improvement, 480 s per seed.
# SEEDS28 env: which seeds (the campaign is split over several gpurun calls).
set -u
out=gpurun_out/${1:-r02tts6}
mkdir -p $out
timeout 3500 python scripts/time_to_hadamard.py --order 28 --population 10000 --fitness f2 --nc 1 --nr 10 \
    --restart-stall 300000 --seeds $SEEDS28 --budget 480 --out $out/tts28.jsonl > /dev/null 2>> $out/err.log
exit 0
