#!/bin/bash
# Which host NUMA node feeds this GPU fastest? PCIe H2D/D2H per node (pinned pages first-touched there).
mkdir -p gpurun_out
{
nvidia-smi topo -m
lscpu | grep -iE "numa|socket|model name"
for d in /sys/devices/system/node/node*; do
  c=$(cat $d/cpulist); echo "== $(basename $d) cpus $c"
  taskset -c $c python tools/pcie_probe.py
done
echo "== no affinity"; python tools/pcie_probe.py
} > gpurun_out/numa_probe.txt 2>&1
cat gpurun_out/numa_probe.txt
