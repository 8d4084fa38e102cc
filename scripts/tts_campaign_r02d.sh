#!/bin/bash
# Round-2 order-28 campaign, the seeds the 240 s protocol left unsolved
# (2, 8, 9, 11, 15) at a 480 s budget (same protocol otherwise: N = 10,000
# pairs, F2, NC = 1, NR = 10, full restarts after 300,000 generations without
# improvement).  The loop is deterministic per seed, so together with
# r02_tts28_restart300k.jsonl this is the 16-seed distribution at 480 s.
set -u
out=gpurun_out/${1:-r02tts28b}
mkdir -p $out
timeout 2700 python scripts/time_to_hadamard.py --order 28 --population 10000 --fitness f2 --nc 1 --nr 10 \
    --restart-stall 300000 --seeds ${SEEDS28:-2 8 9 11 15} --budget 480 --out $out/tts28.jsonl > /dev/null 2>> $out/err.log
exit 0
