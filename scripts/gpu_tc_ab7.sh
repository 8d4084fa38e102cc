#!/bin/bash
tag=${1:-tcab7}
out=gpurun_out/$tag
mkdir -p $out
for f in 0 8 2 4; do
HGA_TC_FLAGS=$f ORDERS=48,52,64 timeout 300 python scripts/tc_sweep.py f$f tc >> $out/sweep.jsonl 2>> $out/sweep.err; echo "sweep rc=$?"
done
