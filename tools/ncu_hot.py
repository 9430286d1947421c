"""Diagnostics: the hottest SASS instructions of an ncu source-page export
(ncu -i rep --page source --csv --print-source sass > f.csv), with their top
stall reasons.    python tools/ncu_hot.py f.csv [n]"""
import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(k, h) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[i_s] or 0) for r in data)
    order = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))
    print(f"total samples {tot:.0f}")
    for k in order[:n]:
        r = data[k]
        s = float(r[i_s] or 0)
        top = sorted(((float(r[c] or 0), h[6:]) for c, h in stall_cols), reverse=True)[:3]
        print(f"{k:5d} {r[0]:>6s} {100 * s / tot:5.1f}%  {r[1][:60]:60s} " +
              " ".join(f"{h}={v:.0f}" for v, h in top if v > 0))


if __name__ == "__main__":
    main()
