#!/bin/bash
# L2-prefetch A/B: GEMM parity subset + cold/warm timings with and without the operand prefetch
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
rm -f gpurun_out/pf_cold_warm.txt
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "gemm" > gpurun_out/pf_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/pf_tests.txt
for pf in 0 1; do BWTA_L2_PREFETCH=$pf timeout 300 python tools/cold_warm.py >> gpurun_out/pf_cold_warm.txt 2>&1; done
BWTA_L2_PREFETCH=0 timeout 300 python bench.py --no-extras --no-cpu > gpurun_out/pf_bench0.json 2>&1
BWTA_L2_PREFETCH=1 timeout 300 python bench.py --no-extras --no-cpu > gpurun_out/pf_bench1.json 2>&1
