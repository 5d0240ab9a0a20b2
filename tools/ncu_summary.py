"""Summarise ncu outputs into profiles/ (launch-list shares, per-kernel DRAM traffic).

Usage: python tools/ncu_summary.py <round-tag> <launches.csv> [name=report.ncu-rep ...]
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from launches import load, num  # noqa: E402


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "").replace("mgrit::", "").replace("(anonymous namespace)::", "")


def launch_summary(path):
    k = load(path)
    agg = OrderedDict()
    total = 0.0
    for (i, name), m in sorted(k.items()):
        t = num(m.get("gpu__time_duration.sum", 0)) / 1000.0
        total += t
        s = agg.setdefault(short(name), [0, 0.0])
        s[0] += 1
        s[1] += t
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    return total, rows, len(k)


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, v = r[0], r[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__block_size"]
    units = r[1]
    res = {}
    for w in want:
        if w in h:
            j = h.index(w)
            res[w] = (v[j], units[j])
    return res


def to_bytes(val, unit):
    x = num(val)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return x * scale


if __name__ == "__main__":
    tag, launches = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    total, rows, nlaunch = launch_summary(launches)
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             f"source: `{os.path.basename(launches)}`, {nlaunch} launches, {total:.1f} us total "
             "(cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (cnt, t) in rows:
        lines.append(f"| `{name}` | {cnt} | {t:.1f} | {100 * t / total:.1f}% |")
    traffic = {}
    if len(sys.argv) > 3:
        lines += ["", "## ncu --set full captures (one launch each)", "",
                  "| capture | duration us | DRAM read MB | DRAM write MB | registers | grid x block |", "|---|---|---|---|---|---|"]
        for spec in sys.argv[3:]:
            key, rep = spec.split("=", 1)
            m = raw_metrics(rep)
            dur = num(m["gpu__time_duration.sum"][0])
            dur_us = dur / 1000 if m["gpu__time_duration.sum"][1] == "ns" else dur
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            traffic[key] = rd + wr
            lines.append(f"| {key} | {dur_us:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                         f"{m.get('launch__registers_per_thread', ('?',))[0]} | "
                         f"{m.get('launch__grid_size', ('?',))[0]} x {m.get('launch__block_size', ('?',))[0]} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        old = json.load(open(p)) if os.path.exists(p) else {}
        old.update(traffic)
        json.dump(old, open(p, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))
