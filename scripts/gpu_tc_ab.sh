#!/bin/bash
# One GPU call: parity suite, then an A/B sweep of the int8 fitness paths at m = 36..64.
tag=${1:-tcab}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
timeout 300 python scripts/tc_sweep.py bal tc > $out/sweep_bal.jsonl 2> $out/sweep_bal.err; echo "bal rc=$?"
HGA_TC_ONEWAIT=1 timeout 300 python scripts/tc_sweep.py onewait tc > $out/sweep_ow.jsonl 2> $out/sweep_ow.err; echo "ow rc=$?"
timeout 300 python scripts/tc_sweep.py popc popc > $out/sweep_popc.jsonl 2> $out/sweep_popc.err; echo "popc rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
