#!/bin/bash
# fused all-gather: peer tests + tile-kernel regression check
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_peer_gpu.py -m gpu -x -q > gpurun_out/p2_tests.txt 2>&1
echo "peer tests exit $?" >> gpurun_out/p2_tests.txt
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py tests/test_dist_gpu.py -m gpu -x -q -k "gemm or r12 or skinny or pack or nshard" >> gpurun_out/p2_tests.txt 2>&1
echo "gemm tests exit $?" >> gpurun_out/p2_tests.txt
timeout 300 python tools/c3_tiles.py > gpurun_out/p2_tiles.txt 2>&1
