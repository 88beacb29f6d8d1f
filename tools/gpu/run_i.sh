#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py -q -m gpu -x -k "gemm or r12 or attention or pack" > gpurun_out/i_tests.txt 2>&1
python tools/c3_tiles.py > gpurun_out/i_tiles.txt 2>&1
for d in 0 24; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/i_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "end_work|period|median" | head -8 >> gpurun_out/i_trace.txt
done
