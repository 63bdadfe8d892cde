"""Summarise tools/prof_tensor_pipe.sh's ncu csv: per kernel class, time and time-weighted tensor-pipe %,
and the level-GEMM aggregate (the north-star '>= 60 % tensor-pipe in the level GEMMs at h >= 1024')."""
import csv
import re
import sys
from collections import defaultdict


def load(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    ker = defaultdict(dict)
    for r in rows[1:]:
        try:
            v = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        ker[int(r[ix["ID"]])][r[ix["Metric Name"]]] = v
        ker[int(r[ix["ID"]])]["name"] = r[ix["Kernel Name"]]
    return ker


def klass(name):
    m = re.match(r"(?:void )?(?:cavs::)?([A-Za-z_0-9]+)", name)
    base = m.group(1) if m else name
    for tag in ("EPI_", "(int)"):
        pass
    e = re.search(r"<\(int\)(\d+)", name) or re.search(r"<(\d+)", name)
    return base + (f"<{e.group(1)}>" if e and base in ("k_rows", "k_tc_level", "k_skinny", "k_persist", "k_gemm_rows") else "")


def main(path):
    ker = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for k, m in ker.items():
        c = klass(m["name"])
        t = m.get("gpu__time_duration.sum", 0.0)
        a = agg[c]
        a[0] += 1
        a[1] += t
        a[2] += t * m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel class':40s} launches  time(us)  share  tensor-pipe% (time-weighted)")
    for c, (n, t, tw) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:40s} {n:8d} {t / 1e3:9.1f} {100 * t / tot:6.1f}% {tw / t if t else 0:8.1f}")
    lev = [a for c, a in agg.items() if c.split("<")[0] in ("k_rows", "k_tc_level", "k_skinny", "k_persist")]
    lt, lw = sum(a[1] for a in lev), sum(a[2] for a in lev)
    print(f"level GEMMs: {lt / 1e3:.1f} us, time-weighted tensor pipe {lw / lt if lt else 0:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
