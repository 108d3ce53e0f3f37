#!/bin/bash
# Round-2 first call: box topology / NUMA (for the per-rank NUMA-local host pools),
# the GPU test suite on the round-1 tree, and a compute-sanitizer memcheck of C1 parity.
mkdir -p gpurun_out/r02a
{
nvidia-smi topo -m
lscpu | head -30
numactl -H 2>/dev/null || echo "no numactl"
ls /sys/devices/system/node/ 2>/dev/null
for d in /sys/bus/pci/devices/*; do
  if [ -f $d/class ] && grep -q 0x0302 $d/class; then echo "$d numa_node=$(cat $d/numa_node)"; fi
done
nvidia-smi --query-gpu=index,pci.bus_id --format=csv
python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"
ldconfig -p | grep -i numa || echo "no libnuma"
free -g
ulimit -l
} > gpurun_out/r02a/probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02a/gpu_tests.log
