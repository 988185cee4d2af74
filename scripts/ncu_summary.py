"""Summarise an ncu report: per kernel time, DRAM bytes, instructions, top stalls."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
def col(name):
    return h.index(name) if name in h else None
want = {
    "time_ms": "gpu__time_duration.sum", "dram_rd": "dram__bytes_read.sum", "dram_wr": "dram__bytes_write.sum",
    "inst": "smsp__inst_executed.sum", "regs": "launch__registers_per_thread",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active", "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1hit": "l1tex__t_sector_hit_rate.pct", "l2hit": "lts__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}
units = rows[1]
stall_cols = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and
              n.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    name = r[col("Kernel Name")].split("(")[0].replace("void ", "")[-45:]
    out = {}
    for k, n in want.items():
        c = col(n)
        if c is not None:
            out[k] = r[c] + ("" if k not in ("dram_rd", "dram_wr", "time_ms") else units[c])
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i].replace(",", "")), h[i].split("stalled_")[-1].replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    print(name, out)
    print("    stalls:", [(n, round(v, 1)) for v, n in st[:6]])
