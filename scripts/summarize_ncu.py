"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/summarize_ncu.py TAG REP [REP ...] [--launches CSV ...] [--workload NAME --rep-for REP]

Writes profiles/<TAG>_ncu.md with, per report: duration, DRAM traffic, pipe utilisations,
issue activity, registers, and the top stall sites; and per launch-list CSV the mean device
time of each kernel (cold-cache, serialised: compare shares, not absolutes).  Also updates
profiles/traffic.json (per-launch DRAM bytes of the dominant kernel per workload), which
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    rows = ncu_csv(rep, "raw")
    h, units, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    metrics = {k: (v[h.index(k)], units[h.index(k)]) for k in KEYS if k in h}
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
            except ValueError:
                pass
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    top = []
    if len(src) > 2:
        hh = src[1]
        si, sc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
        data = [(int(r[si]) if r[si].isdigit() else 0, r[sc].strip()) for r in src[2:] if len(r) > si]
        tot = sum(d[0] for d in data) or 1
        ops = Counter()
        for n, s in data:
            tok = s.split()
            op = (tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")).split(".")[0]
            ops[op] += n
        top = [(op, round(100.0 * n / tot, 1)) for op, n in ops.most_common(12)]
    return name, metrics, stalls, top


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        agg[r[hdr.index("Kernel Name")].split("(")[0]].append(float(r[hdr.index("Metric Value")].replace(",", "")))
    return {k: (len(v), sum(v) / len(v) / 1e3) for k, v in agg.items()}


def main():
    args = sys.argv[1:]
    tag = args.pop(0)
    reps, lcsv, traffic = [], [], {}
    while args:
        a = args.pop(0)
        if a == "--launches":
            lcsv.append(args.pop(0))
        elif a == "--traffic":  # WORKLOAD=REP
            wl, rep = args.pop(0).split("=", 1)
            traffic[wl] = rep
        else:
            reps.append(a)
    out = [f"# ncu summary — {tag}", "",
           "Captured with `ncu --set full --clock-control none --import-source on` (one launch,"
           " ~40 replays) and `ncu --metrics gpu__time_duration.sum` launch lists (cold-cache,"
           " serialised: compare shares, not absolutes).  Regenerate: `python scripts/summarize_ncu.py`.", ""]
    for c in lcsv:
        out += [f"## Launch list `{os.path.basename(c)}`", "", "| kernel | launches | mean µs |", "|---|---|---|"]
        for k, (n, us) in launches(c).items():
            out.append(f"| `{k.strip()}` | {n} | {us:.1f} |")
        out.append("")
    tj_path = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
    for rep in reps:
        name, m, stalls, top = summarize(rep)
        out += [f"## `{os.path.basename(rep)}` — `{name}`", "", "| metric | value |", "|---|---|"]
        for k, (val, unit) in m.items():
            out.append(f"| {k} | {val} {unit} |")
        out += ["", "Warp-stall samples (all warps, incl. idle/waiting roles): " +
                ", ".join(f"{k} {int(v)}" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]), "",
                "Stall samples by opcode (%): " + ", ".join(f"{op} {p}" for op, p in top), ""]
        for wl, r in traffic.items():
            if r == rep:
                rd = float(m["dram__bytes_read.sum"][0]) * (1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1e6)
                wr = float(m["dram__bytes_write.sum"][0]) * (1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1e6)
                tj[wl] = rd + wr
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w").write("\n".join(out) + "\n")
    json.dump(tj, open(tj_path, "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
