#!/bin/bash
# Which role limits the tensor-core fitness kernel: drop one role's work at a time (HGA_TC_FLAGS).
tag=${1:-tcroles}
out=gpurun_out/$tag
mkdir -p $out
for f in 0 2 4 8 6 12 14 0; do
  HGA_TC_FLAGS=$f ORDERS=48,60,64 timeout 300 python scripts/tc_sweep.py flags$f tc >> $out/roles.jsonl 2>> $out/roles.err; echo "flags $f rc=$?"
done
