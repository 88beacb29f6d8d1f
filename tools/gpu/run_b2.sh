#!/bin/bash
# bench: default line, the sharded path at N = 1 through both gathers, peer tests
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peer_gpu.py -m gpu -q > gpurun_out/b2_tests.txt 2>&1
echo "exit $?" >> gpurun_out/b2_tests.txt
timeout 600 python bench.py --no-extras --no-cpu > gpurun_out/b2_default.json 2> gpurun_out/b2_default.err
timeout 600 python bench.py --nshard --gather peer --no-extras --no-cpu > gpurun_out/b2_peer.json 2> gpurun_out/b2_peer.err
timeout 600 python bench.py --nshard --gather nccl --chunks 1 --no-extras --no-cpu > gpurun_out/b2_nccl.json 2> gpurun_out/b2_nccl.err
timeout 600 python bench.py --workload nshard_gemm --nshard --gather peer --no-extras --no-cpu > gpurun_out/b2_c4_peer.json 2> gpurun_out/b2_c4_peer.err
