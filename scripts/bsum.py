"""Summarise bench JSON lines: python scripts/bsum.py gpurun_out/bench*.log"""
import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        k = d.get("kernel_ms_per_launch") or {}
        print(f, "ms/iter %.2f" % d.get("ms_per_step", 0), "value %.3g" % d.get("value", 0),
              " ".join("%s=%.2f" % (a, b) for a, b in sorted(k.items(), key=lambda x: -x[1])[:6]),
              "frac=%s" % (d.get("roofline") or {}).get("frac"))
