#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 7 0; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/j_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | head -22 >> gpurun_out/j_trace.txt
done
