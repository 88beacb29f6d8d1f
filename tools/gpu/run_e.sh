#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/c3_tiles.py > gpurun_out/e_tiles.txt 2>&1
for d in 0 2 7; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/e_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "median|end_work" | head -7 >> gpurun_out/e_trace.txt
done
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py -q -m gpu -x -k "gemm or r12" > gpurun_out/e_tests.txt 2>&1
echo done
