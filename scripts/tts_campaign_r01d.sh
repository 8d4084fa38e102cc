#!/bin/bash
# Round-1 campaign 4: order-20 statistics over 16 seeds (paper section 4.4 setting) and
# order 28 (paper setting, 40,000 matrices) with stall restarts over 12 seeds.
# Also checks the torchrun launch path of bench.py at world size 1.
set -u
mkdir -p gpurun_out/r01d
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 50 --warmup 3 --no-sweep --no-cpu > gpurun_out/r01d/bench_torchrun.json 2> gpurun_out/r01d/bench_torchrun.err
echo "torchrun bench rc=$?"
OUT=gpurun_out/r01d/tts.jsonl
python scripts/time_to_hadamard.py --order 20 --population 1000 --nc 2 --nr 8 --seeds $(seq 0 15) --budget 60 --out $OUT
python scripts/time_to_hadamard.py --order 28 --population 10000 --nc 1 --nr 10 --stall 50000 --seeds $(seq 0 11) --budget 150 --out $OUT
