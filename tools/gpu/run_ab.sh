#!/bin/bash
# A/B of library variants: parity subset on the default lib, C3 tiles + cold/warm per variant lib
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
P=${1:-ab}; shift
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py tests/test_binary_w1a1.py tests/test_attn_prefill.py -m gpu -x -q > gpurun_out/${P}_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/${P}_tests.txt
tail -2 gpurun_out/${P}_tests.txt
for lib in libbwta.so "$@"; do
  echo "=== $lib"
  BWTA_LIB=$lib timeout 300 python tools/c3_tiles.py 2>&1
  BWTA_LIB=$lib timeout 300 python tools/cold_warm.py 2>&1
done > gpurun_out/${P}_tiles.txt
cat gpurun_out/${P}_tiles.txt
