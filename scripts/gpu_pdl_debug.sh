#!/bin/bash
mkdir -p gpurun_out
SKV_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tiny_config_full_parity and 0-8" > gpurun_out/pdl_pytest.txt 2>&1; tail -5 gpurun_out/pdl_pytest.txt
SKV_PDL=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pdl_sanitizer.txt 2>&1; head -60 gpurun_out/pdl_sanitizer.txt
SKV_PDL=1 CUDA_LAUNCH_BLOCKING=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pdl_blocking.txt 2>&1; tail -c 400 gpurun_out/pdl_blocking.txt
