#!/bin/bash
# A/B of the tensor-core fitness piece order + parity + one ncu capture per order.
tag=${1:-tcab2}
out=gpurun_out/$tag
mkdir -p $out
timeout 300 python scripts/tc_sweep.py cf tc > $out/sweep_cf.jsonl 2> $out/sweep_cf.err; echo "cf rc=$?"
HGA_TC_ROWMAJOR=1 timeout 300 python scripts/tc_sweep.py rowmajor tc > $out/sweep_rm.jsonl 2> $out/sweep_rm.err; echo "rm rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
for m in 64 48; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fit_i8_tc -s 2 -c 1 -o $out/fit_tc$m \
    python scripts/prof_tc.py $m 1000000 > $out/ncu_tc$m.log 2>&1; echo "ncu $m rc=$?"
done
