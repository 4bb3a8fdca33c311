"""profiles/ncu_traffic.json from an ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum CSV
of `bench.py --profile-only` (measurement tool): DRAM bytes (read + write) per launch, averaged
over the launches of each kernel, keyed by the names bench.py's kernel table uses.

usage: python tools/traffic_json.py <traffic.csv> <out.json>
"""
import csv
import re
import io
import json
import sys
from collections import defaultdict

NAMES = [(r"masq_gemm_kernel<(\(int\))?0[,>]", "gemm_fwd"), (r"masq_gemm_kernel<(\(int\))?2[,>]", "gemm_loss"),
         (r"masq_gemm_kernel<(\(int\))?3[,>]", "gemm_ref"), (r"masq_gemm_kernel<(\(int\))?5[,>]", "gemm_alpha_i8"),
         ("aquant_bf16_kernel", "aquant"), ("aquant_row_kernel", "aquant"), ("stats_kernel", "stats"),
         ("init_kernel", "init"), ("wcolmax_tma_kernel", "wcolmax"), ("wquant_tma_kernel", "wquant"),
         ("wcolmax_kernel", "wcolmax"), ("wquant_kernel", "wquant"), ("route_scatter_kernel", "route"),
         ("pad_rows_kernel", "pad_rows"), ("gather_rows_kernel", "gather_rows"), ("zgemm_kernel", "zgemm"),
         ("route_kernel", "route")]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(src, dst):
    txt = open(src).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    hdr = rows[0]
    ni, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = defaultdict(float)
    names = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        per[r[ii]] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        names[r[ii]] = r[ni]
    agg = defaultdict(list)
    for i, b in per.items():
        for pat, key in NAMES:
            if re.search(pat, names[i]):
                agg[key].append(b)
                break
    out = {k: sum(v) / len(v) for k, v in agg.items()}
    out["_note"] = ("DRAM bytes (read+write) per launch, averaged over the launches of the profiled step; ncu "
                    f"--metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none on bench.py --profile-only ({src})")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
