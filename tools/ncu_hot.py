"""Top stall-sampled SASS lines of one kernel from `ncu --page source --csv` output (measurement tool)."""
import csv
import sys


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Address" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[wi]) for r in data) or 1.0
    for r in sorted(data, key=lambda r: -f(r[wi]))[:n]:
        print(f"{f(r[wi]) / tot * 100:5.1f}%  {r[si][:120]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
