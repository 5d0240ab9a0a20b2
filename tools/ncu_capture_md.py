"""Summarise `ncu --set full` captures (.ncu-rep) into a markdown table:
time, DRAM bytes and throughput, FP64 pipe and issue utilisation, occupancy,
registers and the top three warp-stall reasons (tools only).
Usage: python tools/ncu_capture_md.py OUT.md TITLE key=path.ncu-rep ..."""
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import to_bytes  # noqa: E402
from launches import num  # noqa: E402

STALL = "smsp__average_warps_issue_stalled_"
SUFFIX = "_per_issue_active.ratio"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (r[2][i], r[1][i]) for i, h in enumerate(r[0])}


def row(key, rep):
    m = raw(rep)
    g = lambda k: num(m[k][0]) if k in m and m[k][0] not in ("", "n/a") else float("nan")  # noqa: E731
    dur = g("gpu__time_duration.sum")
    unit = m["gpu__time_duration.sum"][1]
    dur_us = dur * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    stalls = sorted(((g(k), k[len(STALL):-len(SUFFIX)]) for k in m if k.startswith(STALL) and k.endswith(SUFFIX)
                     and "not_issued" not in k and not k[len(STALL):].startswith(("selected", "not_selected"))), reverse=True)[:3]
    return (f"| {key} | {dur_us:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
            f"{(rd + wr) / (dur_us * 1e-6) / 1e9:.0f} | {g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g('sm__issue_active.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {m.get('launch__registers_per_thread', ('?',))[0]} | "
            f"{m.get('launch__grid_size', ('?',))[0]} x {m.get('launch__block_size', ('?',))[0]} | "
            + ", ".join(f"{n} {v:.2f}" for v, n in stalls) + " |")


def main():
    out, title, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# {title}", "",
             "One launch per capture, `ncu --set full --clock-control none --import-source on` (cold cache, "
             "serialised). Stalls are warps stalled per issued instruction, top three.", "",
             "| capture | us | DRAM read MB | DRAM write MB | DRAM GB/s | FP64 pipe % | issue active % | warps active % "
             "| regs | grid x block | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for spec in specs:
        key, rep = spec.split("=", 1)
        lines.append(row(key, rep))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
