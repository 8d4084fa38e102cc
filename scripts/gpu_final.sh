#!/bin/bash
# Full GPU suite + fitness sweep + bench + tc ncu after the last kernel change.
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 900 python scripts/probe.py --only fitness > $out/fitness_sweep.jsonl 2> $out/fitness_sweep.err; echo "probe rc=$?"
for m in 48 64; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc -s 2 -c 1 -o $out/fit_tc$m \
    python scripts/prof_tc.py $m 1000000 > $out/ncu_tc$m.log 2>&1; echo "ncu $m rc=$?"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; echo "smoke rc=$?"
