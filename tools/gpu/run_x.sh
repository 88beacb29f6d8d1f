#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 7 263 519 1031 1799; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/x_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 60 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "end_work|period" | head -5 >> gpurun_out/x_trace.txt
done
