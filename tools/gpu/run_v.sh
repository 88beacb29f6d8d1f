#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 0 128 7 135; do
  echo "=== BWTA_DBG=$d" >> gpurun_out/v_trace.txt
  BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "end_work|period" | head -4 >> gpurun_out/v_trace.txt
done
