"""Summarise ncu reports / launch lists into profiles/ (text + json)."""
import csv, json, subprocess, sys, io, collections

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
           "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
           "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]

def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = f"{vals[i]} {units[i]}".strip()
    return d

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    out = collections.OrderedDict()
    for r in rows:
        if len(r) == len(hdr) and r != hdr:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out[int(d["ID"])] = (d["Kernel Name"], d["Grid Size"], float(d["Metric Value"]))
    return out

if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "report":
        print(json.dumps(report(path), indent=1))
    else:
        L = launches(path)
        ids = sorted(L)
        last = int(sys.argv[3]) if len(sys.argv) > 3 else len(ids) // 2
        half = ids[-last:]                   # the last step (earlier launches: calibration, warm-up)
        tot = sum(L[i][2] for i in half)
        agg = collections.defaultdict(float)
        print(f"{'id':>4} {'ns':>9} {'share':>6}  kernel (grid)")
        for i in half:
            name, grid, ns = L[i]
            short = name.split("(")[0].replace("void bwta::<unnamed>::", "").replace("bwta::<unnamed>::", "")
            agg[short] += ns
            print(f"{i:4d} {ns:9.0f} {ns / tot:6.1%}  {short} {grid}")
        print(f"total {tot:.0f} ns over {len(half)} launches (ncu: serialized, cold cache)")
        for k, v in sorted(agg.items(), key=lambda x: -x[1]):
            print(f"  {v / tot:6.1%}  {k}")
