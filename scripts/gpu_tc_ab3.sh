#!/bin/bash
tag=${1:-tcab3}
out=gpurun_out/$tag
mkdir -p $out
timeout 300 python scripts/tc_sweep.py chk tc > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
HGA_TC_FLAGS=8 ORDERS=48,60,64 timeout 300 python scripts/tc_sweep.py nochk tc > $out/sweep_nochk.jsonl 2>> $out/sweep.err; echo "nochk rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
