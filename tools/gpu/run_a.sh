#!/bin/bash
# round-2 GPU pass A: parity (new large-size tests first), bench (configs[2] headline), ncu.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_gpu.txt
timeout 900 python -m pytest tests/test_parity_gpu_large.py -q -m gpu -rf > gpurun_out/a_tests_large.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -rf --deselect tests/test_parity_gpu_large.py > gpurun_out/a_tests_all.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/r02_ncu_gemm_n11008 python tools/prof_c3.py 11008 > gpurun_out/a_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/r02_ncu_gemm_n4096 python tools/prof_c3.py 4096 > gpurun_out/a_ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_llama.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/a_ncu3.log 2>&1
echo done
