"""Summarise ncu outputs for profiles/ (measurement tool).

usage:
  python tools/ncu_summary.py rep  <file.ncu-rep>   -> per-kernel key metrics (markdown table)
  python tools/ncu_summary.py launches <launches.csv> -> per-kernel launch count / time share
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
    name_i = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(lbl for k, lbl in KEYS if k in idx) + " |")
    print("|---" * (1 + len(idx)) + "|")
    for r in rows[2:]:
        nm = r[name_i].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        vals = []
        for k, lbl in KEYS:
            if k in idx:
                vals.append(f"{r[idx[k]]} {units[idx[k]]}".strip())
        print(f"| {nm[:60]} | " + " | ".join(vals) + " |")


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ni, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ui = hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        nm = r[ni].split("(")[0].replace("void ", "")
        agg[nm][0] += 1
        agg[nm][1] += ms
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ms (serialised, cold) | share |")
    print("|---|---|---|---|")
    for nm, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {nm[:70]} | {c} | {ms:.3f} | {ms / tot:.3f} |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
