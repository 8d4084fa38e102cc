#!/bin/bash
out=gpurun_out/m44; mkdir -p $out
ORDERS=44 NMAT=500000 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_v2 -s 0 -c 1 -o $out/f2 python scripts/tc_sweep.py x popc > $out/f2.log 2>&1; echo "f2 rc=$?"
ORDERS=44 NMAT=500000 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_v2 -s 13 -c 1 -o $out/f1 python scripts/tc_sweep.py x popc > $out/f1.log 2>&1; echo "f1 rc=$?"
