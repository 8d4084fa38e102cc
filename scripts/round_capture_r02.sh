#!/bin/bash
# Round-2 evidence in one GPU call: GPU tests, bench (both arms), kernel
# launch list, ncu --set full of the generation kernel (k_run_v3) and of the
# round-2 tensor-core fitness kernel (k_fit_i8_tc2) at m = 48 / 64, the
# fitness sweep (probe.py) and phase timing.  Output: gpurun_out/<tag>/.
tag=${1:-r02cap}
out=gpurun_out/$tag
mkdir -p $out
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
  tail -2 $out/pytest_gpu.log
fi
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_run_v3 -s 30 -c 1 -o $out/k_run \
    python bench.py --steps 40 --warmup 3 --no-sweep --no-cpu > $out/ncu_krun.log 2>&1; echo "ncu k_run rc=$?"
for m in 48 64; do
  HGA_FITNESS_TC=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc2 -s 2 -c 1 \
      -o $out/fit_tc$m python scripts/prof_tc.py $m 1000000 > $out/ncu_tc$m.log 2>&1; echo "ncu tc$m rc=$?"
done
timeout 900 python scripts/probe.py --only fitness > $out/fitness_sweep.jsonl 2> $out/fitness_sweep.err; echo "probe rc=$?"
timeout 300 python scripts/phase_timing.py > $out/phase.jsonl 2>&1; echo "phase rc=$?"
