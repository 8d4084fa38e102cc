#!/bin/bash
# Order 36 with the order-28 protocol (40,000 matrices, F2, NC = 1, NR = 12,
# full restarts after 300,000 generations without improvement), 1,200 s per
# seed.  The paper never reached order 36.
set -u
out=gpurun_out/${1:-r02tts36b}
mkdir -p $out
timeout 5200 python scripts/time_to_hadamard.py --order 36 --population 10000 --fitness f2 --nc 1 --nr 12 \
    --restart-stall 300000 --seeds ${SEEDS36:-0 1 2 3} --budget 1200 --out $out/tts36.jsonl > /dev/null 2>> $out/err.log
exit 0
