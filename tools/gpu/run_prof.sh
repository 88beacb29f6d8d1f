#!/bin/bash
# ncu evidence for the current code: --set full of the dominant GEMM (C3 N=11008) and of N=4096,
# plus the launch list (gpu__time_duration) of a short bench run
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
P=${1:-r02m}
export PATH=$PATH:/usr/local/cuda/bin
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/${P}_ncu_gemm_n11008 python tools/prof_c3.py 11008 > gpurun_out/${P}_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/${P}_ncu_gemm_n4096 python tools/prof_c3.py 4096 > gpurun_out/${P}_ncu2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_llama.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/${P}_ncu3.log 2>&1
echo done
