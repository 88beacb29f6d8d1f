#!/bin/bash
# ncu evidence for the current code: --set full of the dominant kernel (the configs[2] grouped GEMM)
# and the launch list (gpu__time_duration) of the bench step's kernels
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
P=${1:-r02q}
export PATH=$PATH:/usr/local/cuda/bin
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/${P}_ncu_gemm_grouped python tools/prof_grouped.py > gpurun_out/${P}_ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_gemm|pack_rows|cc_gemv|gemv' -c 60 --csv --log-file gpurun_out/${P}_launches_llama.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/${P}_ncu3.log 2>&1
echo done
