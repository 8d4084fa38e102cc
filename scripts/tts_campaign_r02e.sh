#!/bin/bash
# Order 32 with the order-28 protocol (40,000 matrices, F2, NC = 1, NR = 12,
# full restarts after 300,000 generations without improvement), 600 s per
# seed; the paper needed 94,923 s for one order-32 matrix.
set -u
out=gpurun_out/${1:-r02tts32}
mkdir -p $out
timeout 3500 python scripts/time_to_hadamard.py --order 32 --population 10000 --fitness f2 --nc 1 --nr 12 \
    --restart-stall 300000 --seeds ${SEEDS32:-0 1 2 3} --budget ${BUDGET32:-600} --out $out/tts32.jsonl > /dev/null 2>> $out/err.log
exit 0
