#!/bin/bash
# 512-K stage A/B: parity (large C3 / configs[4] / grouped / R12 + GEMM tests) with BWTA_KS512=1, then timings both ways
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
BWTA_KS512=1 timeout 300 python -m pytest tests/test_parity_gpu_large.py -m gpu -x -q -k "grouped" > gpurun_out/ks_tests0.txt 2>&1
echo "grouped test exit $?"; tail -2 gpurun_out/ks_tests0.txt
BWTA_KS512=1 timeout 600 python -m pytest tests/test_parity_gpu_large.py tests/test_parity_gpu.py -m gpu -x -q -k "gemm or r12 or configs" > gpurun_out/ks_tests.txt 2>&1
echo "tests exit $?"; tail -2 gpurun_out/ks_tests.txt
for v in 0 1; do echo "== KS512=$v"; BWTA_KS512=$v timeout 120 python tools/cold_warm.py 2>&1 | grep -v "in-graph"; BWTA_KS512=$v timeout 120 python tools/grouped_ab.py 2>&1 | head -2; done
