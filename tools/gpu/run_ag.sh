#!/bin/bash
# tile-kernel change check: GEMM/attention parity subset, C3 tile timings, cold/warm, bench line
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
P=${1:-ag}
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_large.py tests/test_binary_w1a1.py -m gpu -x -q > gpurun_out/${P}_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/${P}_tests.txt
timeout 300 python tools/c3_tiles.py > gpurun_out/${P}_tiles.txt 2>&1
timeout 300 python tools/cold_warm.py > gpurun_out/${P}_cold_warm.txt 2>&1
timeout 300 python bench.py --no-extras --no-cpu > gpurun_out/${P}_bench.json 2>&1
python - "$P" <<'PY'
import json, sys
p = sys.argv[1]
print(open(f"gpurun_out/{p}_tests.txt").read().strip().splitlines()[-2:])
print(open(f"gpurun_out/{p}_tiles.txt").read())
print(open(f"gpurun_out/{p}_cold_warm.txt").read())
try:
    d = json.loads(open(f"gpurun_out/{p}_bench.json").read().strip().splitlines()[-1])
    print(d["value"], d["ms_per_step"], d["per_op_us"], d.get("in_step_us"), d["roofline"]["frac"])
except Exception as e:
    print("bench parse failed", e, open(f"gpurun_out/{p}_bench.json").read()[-2000:])
PY
