"""Summarise a round's GPU captures into profiles/ (tracked).

    python scripts/summarize_profiles.py --tag r01 --bench gpurun_out/bench43.log \
        --launches gpurun_out/launches43.csv --rep gpurun_out/prof43.ncu-rep --config c2

Writes profiles/<tag>_bench_<config>.json (the bench line), <tag>_launches_<config>.md (per
kernel: launches, mean device time, share, DRAM bytes per launch — cold-cache, serialised),
<tag>_ncu_<kernel>.md (the --set full capture: key metrics + top stall lines) and
traffic_<config>.json (DRAM bytes per launch per kernel, read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("sfv::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return n.strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        per[d["ID"]]["name"] = d["Kernel Name"]
        try:
            per[d["ID"]]["m"][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    agg = defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    for v in per.values():
        k = short(v["name"])
        m = v["m"]
        a = agg[k]
        a["n"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6, "ns": 1.0, "us": 1e3, "ms": 1e6, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    res = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = {}
        for k, u, v in zip(h, units, r):
            if u in scale and v not in ("", "n/a"):
                try:
                    v = repr(float(v.replace(",", "")) * scale[u])
                except ValueError:
                    pass
            d[k] = v
        res.append(d)
    return res


KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--bench")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, f"traffic_{args.config}.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    traffic.setdefault("dram_bytes_per_launch", {})
    if args.bench:
        line = [l for l in open(args.bench) if l.startswith("{")][-1]
        json.dump(json.loads(line), open(os.path.join(prof, f"{args.tag}_bench_{args.config}.json"), "w"), indent=1)
    if args.launches:
        agg = launches(args.launches)
        tot = sum(a["ns"] for a in agg.values()) or 1.0
        lines = [f"# {args.tag} launch list ({args.config}) — ncu gpu__time_duration, cold-cache, serialised",
                 "", "| kernel | launches | mean us | share | DRAM MB read/launch | DRAM MB written/launch |",
                 "|---|---:|---:|---:|---:|---:|"]
        for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
            lines.append(f"| {k} | {a['n']} | {a['ns'] / a['n'] / 1e3:.1f} | {100 * a['ns'] / tot:.1f}% | "
                         f"{a['rd'] / a['n'] / 1e6:.1f} | {a['wr'] / a['n'] / 1e6:.1f} |")
            base = k.split("<")[0]
            if a["rd"] > 0 and base not in traffic["dram_bytes_per_launch"]:
                traffic["dram_bytes_per_launch"][base] = (a["rd"] + a["wr"]) / a["n"]
        open(os.path.join(prof, f"{args.tag}_launches_{args.config}.md"), "w").write("\n".join(lines) + "\n")
    if args.rep:
        import ncu_lines  # noqa: F401  (same directory)
        for d in raw_metrics(args.rep):
            k = short(d["Kernel Name"])
            base = k.split("<")[0]
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
            traffic["dram_bytes_per_launch"][base] = rd + wr
            out = [f"# {args.tag} ncu --set full: {k} ({args.config})", "",
                   f"source: `{os.path.basename(args.rep)}` (gpurun_out, not tracked); cold-cache, clocks not locked", "",
                   "| metric | value |", "|---|---:|"]
            for key, label in KEYS:
                if key in d and d[key] not in ("", None):
                    out.append(f"| {label} (`{key}`) | {d[key]} |")
            stalls = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), args.rep, base, "20"],
                                    capture_output=True, text=True).stdout
            out += ["", "Top source lines by warp-stall samples (scripts/ncu_lines.py):", "", "```", stalls.rstrip(), "```"]
            open(os.path.join(prof, f"{args.tag}_ncu_{base}.md"), "w").write("\n".join(out) + "\n")
    traffic["note"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu, cold cache)"
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
