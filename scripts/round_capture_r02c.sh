#!/bin/bash
# Last round-2 refresh: GPU tests, smoke, bench (both arms), host-step A/B,
# launch list of the bench.  Output: gpurun_out/<tag>/.
tag=${1:-r02g}
out=gpurun_out/$tag
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout 300 python scripts/e2e_bits_ab.py > $out/e2e_ab.log 2>&1; echo "e2e ab rc=$?"
timeout 300 python scripts/multi_variant_ab.py > $out/multi_variant_ab.jsonl 2>&1; echo "multi-variant ab rc=$?"
timeout 300 python scripts/e2e_same_steps.py 20 > $out/e2e_same.log 2>&1; echo "e2e same rc=$?"
timeout 300 python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu > $out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
