#!/bin/bash
# PCIe end-to-end rate vs the NUMA node the pinned host buffers live on
mkdir -p gpurun_out
nvidia-smi topo -m 2>&1 | head -8
lscpu | grep -i -E "numa|socket|model name" 
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/numa_node 2>/dev/null
for node in $(ls -d /sys/devices/system/node/node* | sed 's/.*node//'); do
  cpus=$(cat /sys/devices/system/node/node$node/cpulist)
  HB_PIPE_CHUNK=$((1<<21)) timeout 300 taskset -c $cpus python bench.py --steps 10 --warmup 3 --no-resnet --no-cpu-baseline > gpurun_out/e2e_node$node.json 2>gpurun_out/e2e_node$node.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_node$node.json'));print('node $node cpus $cpus', d['e2e']['value'])"
  grep "per-step" gpurun_out/e2e_node$node.err
done
