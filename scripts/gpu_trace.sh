#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py > gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt | tail -20
