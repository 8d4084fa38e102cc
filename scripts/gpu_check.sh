#!/bin/bash
# One GPU round trip: parity tests, phase timing, fitness sweep, short bench.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
tag=${1:-check}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 300 python scripts/phase_timing.py > $out/phase_timing.jsonl 2> $out/phase_timing.err
echo "phase rc=$?"
timeout 600 python scripts/probe.py --only fitness --quick > $out/fitness_sweep.jsonl 2> $out/fitness_sweep.err
echo "probe rc=$?"
timeout 600 python bench.py --steps 300 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$?"
cat $out/bench.json | cut -c1-600
