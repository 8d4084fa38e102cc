#!/bin/bash
# pipe probes (POPC, ALU, int8 tcgen05 at 128x256x32 and 64x64x32) + ncu of the
# round-2 tensor-core fitness kernel.  Output: gpurun_out/$1/
out=gpurun_out/${1:-tc2p}
mkdir -p $out
[ -n "$PIPES" ] && timeout 300 python scripts/probe.py --only pipes > $out/pipes.jsonl 2>&1
export HGA_FITNESS_TC=2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc2 -s 2 -c 1 \
  -o $out/tc2_48 python scripts/prof_tc.py 48 1000000 > $out/ncu48.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc2 -s 2 -c 1 \
  -o $out/tc2_60 python scripts/prof_tc.py 60 1000000 > $out/ncu60.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc2 -s 2 -c 1 \
  -o $out/tc2_56 python scripts/prof_tc.py 56 1000000 > $out/ncu56.log 2>&1
tail -n 2 $out/ncu*.log
