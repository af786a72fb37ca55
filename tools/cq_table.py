"""Summarise gpurun_out/cq_launches_<c>.csv (tools/cq_launches.sh) as per-launch rows + total."""
import csv, io, sys
for c in sys.argv[1:]:
    txt = open(f"gpurun_out/cq_launches_{c}.csv").read()
    rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[1:]:
        d.setdefault(r[ii], {"k": r[ki][:44]})[r[mi]] = r[vi]
    tot = 0.0
    for v in d.values():
        t = float(v["gpu__time_duration.sum"]) / 1e6
        tot += t
        print(c, v["k"], v.get("launch__grid_size"), v.get("launch__cluster_dim_x"), round(t, 3))
    print(c, "total", round(tot, 2))
