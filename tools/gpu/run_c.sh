#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for d in 0 1 2 3 4 5 6 7; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/c_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "median|end_work|epi_tfull" | head -12 >> gpurun_out/c_trace.txt
done
for d in 0 1 2 3; do
  echo "=== 4096 BWTA_DBG=$d" >> gpurun_out/c_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 4096 2>&1 | grep -E "median|end_work|epi_tfull" | head -12 >> gpurun_out/c_trace.txt
done
echo done
