#!/bin/bash
mkdir -p gpurun_out
free -g > gpurun_out/probe.txt; nproc >> gpurun_out/probe.txt; nvidia-smi topo -m >> gpurun_out/probe.txt 2>&1
timeout 120 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/tma_host_probe scripts/probes/tma_host_probe.cu && ./scripts/probes/tma_host_probe >> gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
