#!/bin/bash
tag=${1:-tcab5}
out=gpurun_out/$tag
mkdir -p $out
timeout 300 python scripts/tc_sweep.py runA tc > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
timeout 300 python scripts/tc_sweep.py runB tc >> $out/sweep.jsonl 2>> $out/sweep.err; echo "sweep rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fitness or tensor" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
