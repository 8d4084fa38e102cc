#!/bin/bash
# A/B of the tensor-core fitness unit size kB (MMA pairs per pipeline unit): 2 (built) vs 1 / 4 (variant libraries).
tag=${1:-tckb}
out=gpurun_out/$tag
mkdir -p $out
L=paper_2208_14961_b200/libhga.so
cp $L /tmp/libhga_kb2.so
for kb in 2 4; do
  cp /tmp/libhga_kb2.so $L; [ $kb != 2 ] && cp paper_2208_14961_b200/variants/libhga_kb$kb.so $L
  timeout 300 python scripts/tc_sweep.py kb$kb tc >> $out/sweep.jsonl 2>> $out/sweep.err; echo "kb$kb rc=$?"
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tensor or both" > $out/pytest_kb$kb.log 2>&1; tail -1 $out/pytest_kb$kb.log
done
cp /tmp/libhga_kb2.so $L
