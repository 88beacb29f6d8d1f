#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
timeout 600 python bench.py --nshard --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/aj_nshard.json 2> gpurun_out/aj_nshard.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_smoke.py > gpurun_out/aj_san_$tool.txt 2>&1
done
cat > /tmp/prof_qkv.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
x = gen.activations((4096, 768), 1).cuda(); w = gen.weights(2304, 768, 2).cuda()
a = B.bwta_pack_act(x, 1.6); wp = B.bwta_pack_weight(w)
for _ in range(3):
    B.bwta_gemm_pack_qkv(a, wp, None, 0.01, 32, 128, 12, 64, (0.5, 0.5, 0.5))
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -f -o gpurun_out/r02_ncu_gemm_pack_qkv python /tmp/prof_qkv.py > gpurun_out/aj_ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_|pack_|gemv' -s 9 --csv --log-file gpurun_out/r02_launches_llama.csv python tools/prof_llama.py > gpurun_out/aj_ncu2.log 2>&1
echo done
