#!/bin/bash
cd "$(dirname "$0")/../.."
for d in 0 16; do
  echo "dbg=$d $(BWTA_DBG=$d timeout 120 python tools/attn_bench.py 2>&1 | head -2 | tr '\n' ' ')" >> gpurun_out/s_attn.txt
done
