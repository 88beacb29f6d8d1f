#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 0 1 2 3 4 8 12 15; do
  echo "dbg=$d $(BWTA_DBG=$d timeout 120 python tools/attn_bench.py 2>&1 | head -1)" >> gpurun_out/p_attn.txt
done
