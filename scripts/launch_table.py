"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if r and r[0] == "ID")
idx = {n: i for i, n in enumerate(h)}
agg = collections.OrderedDict()
for r in rows[rows.index(h) + 1:]:
    if len(r) != len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("p2g::", "").replace("<unnamed>::", "")
    t = float(r[idx["Metric Value"]].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[idx["Metric Unit"]], 1e-6)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'ms/launch':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:48]:48s} {n:8d} {t:10.3f} {t / n:10.4f} {100 * t / tot:6.1f}%")
print(f"{'TOTAL':48s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
