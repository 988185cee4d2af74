"""Top CUDA source lines of one kernel in an ncu report, by warp-stall samples.
usage: ncu_lines.py report.ncu-rep kernel_regex [n]"""
import csv, io, os, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
data, fname, h = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        h = r
        si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        continue
    if h is None or not r[0]:
        continue
    try:
        data.append((float(r[si] or 0), float(r[ii] or 0), f"{fname}:{r[0]}", r[1].strip()[:80]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
toti = sum(d[1] for d in data) or 1.0
for s, inst, where, text in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% stall {100 * inst / toti:5.1f}% inst  {where:<22} {text}")
