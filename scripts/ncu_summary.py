"""Summarise an ncu report: key metrics + stall reasons + top stalled SASS (dev aid).
    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [--source]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("kernel:", d.get("Kernel Name", "")[:90])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {units[hdr.index(k)]}")
    st = {k: float(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
          not k.endswith("not_issued") and v.replace('.', '', 1).isdigit()}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1]} {100*v/tot:.0f}%" for k, v in
                                 sorted(st.items(), key=lambda x: -x[1])[:7]))
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    h = r[1]; data = r[2:]
    si = h.index("Warp Stall Sampling (All Samples)")
    c = Counter(); n = Counter()
    for x in data:
        if not x[si].isdigit(): continue
        toks = x[1].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        c[op.split('.')[0]] += int(x[si]); n[op.split('.')[0]] += 1
    print("  samples by opcode:", c.most_common(10))
    print("  static count by opcode:", n.most_common(10))
