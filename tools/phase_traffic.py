"""Fold gpurun_out/traffic_<cfg>_<key>.csv (tools/gpu_phase_traffic.sh) into
profiles/ncu_traffic.json (DRAM bytes per phase launch, summed over the
phase's kernels) and profiles/<tag>_phase_traffic.md.  Usage:
python tools/phase_traffic.py r01f"""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import to_bytes  # noqa: E402


def phase_rows(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = {}
    for r in csv.DictReader(lines[start:]):
        d = per.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"].startswith("dram__"):
            d[r["Metric Name"]] = to_bytes(r["Metric Value"], r["Metric Unit"])
        else:
            d["us"] = v / (1e3 if r["Metric Unit"] in ("ns", "nsecond") else 1.0)
    return list(per.values())


def main(tag):
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tj))
    md = [f"# {tag}: DRAM traffic of whole fused phases (ncu, cold cache, serialised)", "",
          "Each row sums every kernel of one phase launch (`tools/gpu_phase_traffic.sh`, "
          "`tools/profile_phase.py`); bench.py reports it as the roofline `traffic`.", "",
          "| config:phase | kernels | DRAM read MB | DRAM write MB | ncu us |", "|---|---|---|---|---|"]
    for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "traffic_*.csv"))):
        base = os.path.basename(path)[len("traffic_"):-4]
        cfg, key = (base.split("_L", 1)[0], "L" + base.split("_L", 1)[1])
        rows = phase_rows(path)
        if not rows:
            continue
        rd = sum(r.get("dram__bytes_read.sum", 0.0) for r in rows)
        wr = sum(r.get("dram__bytes_write.sum", 0.0) for r in rows)
        us = sum(r.get("us", 0.0) for r in rows)
        traffic[f"{cfg}:{key}"] = rd + wr
        names = sorted({r["kernel"] for r in rows})
        md.append(f"| {cfg}:{key} | {len(rows)} ({', '.join(names)}) | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {us:.1f} |")
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_phase_traffic.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01f")
