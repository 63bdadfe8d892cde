"""Summarise a round's ncu captures (gpurun_out/) into committed profiles/ files.

    python tools/summarize_profiles.py --round r01 [--src gpurun_out]

Writes profiles/<round>_launches.csv (trimmed launch list), profiles/<round>_summary.md
(per-kernel-class time shares of one step, ncu metrics of the captured level kernels) and
profiles/traffic.json (DRAM bytes per launch of the level kernels, read by bench.py).
"""
import argparse
import csv
import json
import os
import re
import subprocess
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kclass(name):
    n = name
    if "k_tc_level" in n:
        m = re.search(r"k_tc_level<\(int\)(\d+), \(int\)(\d+), \(int\)(\d+)>", n) or \
            re.search(r"k_tc_level<(\d+), (\d+), (\d+)>", n)
        epi = {"0": "fwd", "1": "xproj", "2": "bwd", "3": "fc_fwd", "4": "fc_xproj", "5": "fc_bwd", "6": "dx"}
        if m:
            return f"tc_level[{epi.get(m.group(1), m.group(1))},CL={m.group(3)}]"
        return "tc_level"
    if "k_persist" in n:
        m = re.search(r"k_persist<(?:\(int\))?(\d+)", n)
        return "persist[" + {"0": "fwd", "2": "bwd", "3": "fc_fwd", "5": "fc_bwd"}.get(m.group(1) if m else "", "?") + "]"
    if "k_gemm_rows" in n:
        m = re.search(r"k_gemm_rows<(?:\(int\))?(\d+)", n)
        return "gemm_rows[" + {"1": "xproj", "4": "fc_xproj", "6": "dx"}.get(m.group(1) if m else "", m.group(1) if m else "?") + "]"
    if "k_skinny" in n:
        m = re.search(r"k_skinny<[^,]+, (?:\(int\))?(\d+), (?:\(int\))?(\d+)", n)
        return "skinny[" + ("fwd" if m and m.group(2) == "0" else "bwd") + "]"
    if "k_rows" in n:
        m = re.search(r"k_rows<(?:\(int\))?(\d+)", n)
        return "rows[" + {"0": "fwd", "2": "bwd", "3": "fc_fwd", "5": "fc_bwd"}.get(m.group(1) if m else "", "?") + "]"
    for k in ("k_lazy", "k_tc_typeII", "k_graph_sched", "k_level_offsets", "k_graph_levels", "k_level_hist",
              "k_level_scan", "k_level_rank", "k_build_maps",
              "k_prep", "k_pull", "k_roots", "k_colsum", "k_pack"):
        if k in n:
            return k
    return "other:" + n[:40]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((int(d["ID"]), d["Kernel Name"], d["Grid Size"], d["Block Size"], float(d["Metric Value"])))
    return out


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--config", default="cfg4:bf16")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    L = launches(os.path.join(a.src, "launches.csv"))
    # one step = from the 2nd schedule launch (warm-up excluded) to the next one
    starts = [i for i, r in enumerate(L) if "k_graph_sched" in r[1] or "k_graph_levels" in r[1]]
    s0 = starts[1] if len(starts) > 1 else 0
    s1 = starts[2] if len(starts) > 2 else len(L)
    step = [r for r in L[s0:s1] if not r[1].startswith("void at::")]
    with open(os.path.join(prof, f"{a.round}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "class", "grid", "block", "gpu_time_ns"])
        for r in L:
            w.writerow([r[0], r[1][:120], kclass(r[1]), r[2], r[3], r[4]])
    tot = sum(r[4] for r in step)
    agg = OrderedDict()
    for r in step:
        c = kclass(r[1])
        t, n = agg.get(c, (0.0, 0))
        agg[c] = (t + r[4], n + 1)
    lines = [f"# {a.round} profile summary ({a.config}, one training step, ncu launch list)", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` launch list of "
             "`bench.py --steps 2 --warmup 1 --pool 2`; cold-cache and serialised, so compare SHARES, "
             "not absolutes (bench.py's CUDA-event phase times are the measured numbers).", "",
             f"Kernels in the step: {len(step)}; serialised kernel time {tot / 1e3:.1f} us.", "",
             "| kernel class | launches | serialised us | share |", "|---|---|---|---|"]
    for c, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {c} | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    # full capture of the level kernels
    traffic = {}
    reps = [os.path.join(a.src, r) for r in ("levels.ncu-rep", "persist.ncu-rep", "rows.ncu-rep", "cfg5.ncu-rep")]
    for rep in [r for r in reps if os.path.exists(r)]:
        hdr, data = raw_metrics(rep)
        ix = {n: i for i, n in enumerate(hdr)}

        def g(r, n):
            try:
                return float(r[ix[n]])
            except Exception:
                return float("nan")
        lines += ["", f"## ncu --set full: {os.path.basename(rep)} (warm caches, `--cache-control none`)", "",
                  "| kernel | grid | us | DRAM read MB | DRAM write MB | L2 hit % | tensor pipe % | issued IPC | regs |",
                  "|---|---|---|---|---|---|---|---|---|"]
        per = defaultdict(list)
        for r in data:
            name = r[ix["Kernel Name"]]
            c = kclass(name)
            us = g(r, "gpu__time_duration.sum") / 1e3 if g(r, "gpu__time_duration.sum") > 1000 else g(r, "gpu__time_duration.sum")
            rd = g(r, "dram__bytes_read.sum")
            wr = g(r, "dram__bytes_write.sum")
            lines.append(f"| {c} | {r[ix['launch__grid_size']] if 'launch__grid_size' in ix else ''} | {us:.2f} | "
                         f"{rd:.3f} | {wr:.3f} | {g(r, 'lts__t_sector_hit_rate.pct'):.1f} | "
                         f"{g(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.2f} | "
                         f"{g(r, 'sm__inst_issued.avg.per_cycle_active'):.2f} | "
                         f"{g(r, 'launch__registers_per_thread'):.0f} |")
            per[c].append((rd + wr) * 1e6)
        fwd = per.get("tc_level[fwd,CL=4]", []) + per.get("skinny[fwd]", []) + per.get("persist[fwd]", [])
        bwd = per.get("tc_level[bwd,CL=4]", []) + per.get("skinny[bwd]", []) + per.get("persist[bwd]", [])
        lazy = per.get("k_lazy", []) or per.get("k_tc_typeII", [])
        if fwd:
            traffic[f"{a.config}:fwd_levels"] = sum(fwd) / len(fwd)
        if bwd:
            traffic[f"{a.config}:bwd_levels"] = sum(bwd) / len(bwd)
        if lazy:
            traffic[f"{a.config}:lazy"] = sum(lazy) / len(lazy)
        lines += ["", "DRAM units as reported by ncu (MB).  traffic.json holds bytes per launch, averaged over "
                  "the captured launches of each pass."]
    bj = os.path.join(a.src, "bench.json")
    if os.path.exists(bj):
        try:
            b = json.loads(open(bj).read().strip().splitlines()[-1])
            lines += ["", "## bench line of the same round (no profiler attached)", "", "```", json.dumps(b, indent=1)[:6000], "```"]
            json.dump(b, open(os.path.join(prof, f"{a.round}_bench.json"), "w"), indent=1)
        except Exception as e:  # noqa: BLE001
            lines += ["", f"(bench.json unreadable: {e})"]
    b5 = os.path.join(a.src, "bench_cfg5.json")
    if os.path.exists(b5):
        try:
            b = json.loads(open(b5).read().strip().splitlines()[-1])
            json.dump(b, open(os.path.join(prof, f"{a.round}_bench_cfg5.json"), "w"), indent=1)
            lines += ["", "## cfg5 bench line (Tree-FC h = 2048, no profiler attached)", "", "```",
                      json.dumps({k: b[k] for k in ("value", "unit", "ms_per_step", "roofline", "phases") if k in b},
                                 indent=1)[:4000], "```"]
        except Exception as e:  # noqa: BLE001
            lines += ["", f"(bench_cfg5.json unreadable: {e})"]
    open(os.path.join(prof, f"{a.round}_summary.md"), "w").write("\n".join(lines) + "\n")
    tp = os.path.join(prof, "traffic.json")
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old.update(traffic)
    json.dump(old, open(tp, "w"), indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
