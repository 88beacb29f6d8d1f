#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dist_gpu.py -q -m gpu -rf > gpurun_out/b_tests_dist.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -rf -x > gpurun_out/b_tests_all.txt 2>&1
export PATH=$PATH:/usr/local/cuda/bin
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_smoke.py > gpurun_out/b_san_$tool.txt 2>&1
done
BWTA_LIB=libbwta_trace.so timeout 300 python tools/trace_gemm.py 2048 4096 11008 > gpurun_out/b_trace_11008.txt 2>&1
BWTA_LIB=libbwta_trace.so timeout 300 python tools/trace_gemm.py 2048 4096 4096 > gpurun_out/b_trace_4096.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_|pack_|gemv' -s 9 --csv --log-file gpurun_out/r02_launches_llama.csv python tools/prof_llama.py > gpurun_out/b_ncu_l.log 2>&1
echo done
