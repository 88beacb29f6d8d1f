for d in 0 1 2; do echo "== BWTA_TC_DBG=$d"; BWTA_TC_DBG=$d BWTA_LIB=libbwta_trace.so timeout 120 python tools/trace_gemm.py 256 4096 256 2>&1 | grep -E "^  (mma|tma) "; done
