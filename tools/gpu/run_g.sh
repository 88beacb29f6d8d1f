#!/bin/bash
cd "$(dirname "$0")/../.."
for t in 192,2 128,2 64,2 192,1 128,1; do
for d in 5 7; do
  echo "=== tile $t BWTA_DBG=$d" >> gpurun_out/g_trace.txt
  BWTA_TILE=$t BWTA_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 2048 4096 11008 2>&1 | grep -E "mma_bready period|end_work" | head -2 >> gpurun_out/g_trace.txt
done
done
