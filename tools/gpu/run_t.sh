#!/bin/bash
# tile-kernel change check: GEMM parity subset + C3 tile timings
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py -m gpu -x -q -k "gemm or r12 or skinny or pack" > gpurun_out/t_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/t_tests.txt
timeout 300 python tools/c3_tiles.py > gpurun_out/t_tiles.txt 2>&1
