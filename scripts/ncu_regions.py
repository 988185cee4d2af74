"""Aggregate an ncu source page (--print-source cuda,sass) of one kernel by
line ranges of one file: warp-stall samples, executed instructions and
shared-memory wavefronts per region.
usage: ncu_regions.py report.ncu-rep kernel_regex file.cu a-b:name [a-b:name ...]"""
import collections, csv, io, os, subprocess, sys

rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
regions = []
for spec in sys.argv[4:]:
    rng, name = spec.split(":", 1)
    a, b = rng.split("-")
    regions.append((int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
cur, h = "?", None
acc = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
tot = [0.0, 0.0, 0.0, 0.0]
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        h = r
        ix = [h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"),
              h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")]
        continue
    if h is None or not r[0].isdigit():
        continue
    try:
        v = [float(r[i] or 0) for i in ix]
    except (ValueError, IndexError):
        continue
    ln = int(r[0])
    name = "other files" if cur != fname else next((n for a, b, n in regions if a <= ln <= b), f"{fname}: rest")
    for j in range(4):
        acc[name][j] += v[j]
        tot[j] += v[j]
print(f"{'region':34s} {'stall%':>7s} {'inst%':>7s} {'smemWF%':>8s} {'excessWF%':>9s}   inst/launch")
for name, v in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{name:34s} {100*v[0]/max(tot[0],1):7.1f} {100*v[1]/max(tot[1],1):7.1f} {100*v[2]/max(tot[2],1):8.1f} "
          f"{100*v[3]/max(tot[2],1):9.1f}   {v[1]:.3e}")
print(f"total: inst {tot[1]:.4e}, shared wavefronts {tot[2]:.4e} (excessive {tot[3]:.4e})")
