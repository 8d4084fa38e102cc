#!/bin/bash
# A/B: int8 XOR+POPC fitness and generation loop after a code change; parity suite; short bench.
tag=${1:-chains}
out=gpurun_out/$tag
mkdir -p $out
ORDERS=16,20,28,32,36,40,44,48 timeout 300 python scripts/tc_sweep.py popc popc > $out/sweep_popc.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
timeout 300 python scripts/phase_timing.py > $out/phase.jsonl 2> $out/phase.err; echo "phase rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
