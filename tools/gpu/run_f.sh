#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 0 8 16 24; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/f_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "median|end_work" | head -7 >> gpurun_out/f_trace.txt
done
