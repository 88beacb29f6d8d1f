#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py -q -m gpu -x -k "gemm or r12" > gpurun_out/am_tests.txt 2>&1
BWTA_NACC=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py -q -m gpu -x -k "gemm or r12" >> gpurun_out/am_tests.txt 2>&1
python tools/c3_tiles.py > gpurun_out/am_tiles2.txt 2>&1
BWTA_NACC=1 python tools/c3_tiles.py > gpurun_out/am_tiles1.txt 2>&1
