#!/bin/bash
# Final round-2 evidence in one GPU call: GPU tests, smoke, bench (both arms),
# launch list of the bench, ncu --set full of the generation kernel, the
# host-state step A/B (bit stream vs int8) and its launch list, launch-cost
# probe, fitness sweep, phase timing.  Output: gpurun_out/<tag>/.
# (The tensor-core fitness kernel did not change since the r02 capture.)
tag=${1:-r02f}
out=gpurun_out/$tag
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout 300 python scripts/e2e_bits_ab.py > $out/e2e_ab.log 2>&1; echo "e2e ab rc=$?"
timeout 300 python scripts/launch_cost.py > $out/launch_cost.jsonl 2>&1; echo "launch cost rc=$?"
timeout 300 python scripts/phase_timing.py > $out/phase.jsonl 2>&1; echo "phase rc=$?"
timeout 900 python scripts/probe.py --only fitness > $out/fitness_sweep.jsonl 2> $out/fitness_sweep.err; echo "probe rc=$?"
timeout 300 python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu > $out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_run_v3 -s 30 -c 1 -o $out/k_run \
    python bench.py --steps 40 --warmup 3 --no-sweep --no-cpu > $out/ncu_krun.log 2>&1; echo "ncu k_run rc=$?"
timeout 120 python scripts/e2e_steps.py 5 > $out/e2e_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/e2e_launches.csv \
    python scripts/e2e_steps.py 5 > $out/ncu_e2e.log 2>&1; echo "ncu e2e rc=$?"
