"""Summarise an ncu --csv launch list (gpu__time_duration etc.) per kernel."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    out = {}
    for r in rows[hi + 1:]:
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        out.setdefault(key, {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
    return out


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return 0.0


if __name__ == "__main__":
    k = load(sys.argv[1])
    tot = 0.0
    for (i, name), m in sorted(k.items()):
        t = num(m.get("gpu__time_duration.sum", 0)) / 1000
        tot += t
        dram = (num(m.get("dram__bytes_read.sum", 0)) + num(m.get("dram__bytes_write.sum", 0))) / 1e6
        print(f"{i:3d} {name[:60]:60s} grid={m.get('launch__grid_size')} blk={m.get('launch__block_size')} "
              f"regs={m.get('launch__registers_per_thread')} t={t:8.1f}us dram={dram:8.1f}MB "
              f"{dram / max(t, 1e-9) * 1e-3:6.2f}TB/s")
    print(f"total {tot:.1f} us")
