#!/bin/bash
# Host pack/unpack throughput and PCIe copy rates on the GPU box.
out=gpurun_out/${1:-hpp}; mkdir -p $out
lscpu > $out/lscpu.txt 2>&1
g++ -O3 -mavx2 -fopenmp scripts/host_pack_probe.cpp -o /tmp/hpp && /tmp/hpp > $out/host_pack.jsonl 2>&1
python scripts/pcie_probe.py > $out/pcie.txt 2>&1
cat $out/host_pack.jsonl $out/pcie.txt; grep -i "model name\|^CPU(s)\|Thread\|Core\|Socket\|L3\|NUMA" $out/lscpu.txt
