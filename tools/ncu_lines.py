"""Diagnostics: per-source-line stall samples and instruction counts of an ncu
source-page export (ncu -i rep --page source --csv --print-source cuda,sass).
    python tools/ncu_lines.py f.csv [n]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[2]
    i_e = hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(k, h) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    lines, fname = {}, None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0]:
            try:
                ln = int(r[0])
            except ValueError:
                continue
            if len(r) <= i_e:
                continue
            a = lines.setdefault((fname, ln), [r[1], 0.0, 0.0, {}])
            a[1] += f(r[i_e])
            a[2] += f(r[i_s])
            for c, h in stall_cols:
                a[3][h[6:]] = a[3].get(h[6:], 0.0) + f(r[c])
    tot = sum(v[2] for v in lines.values())
    print("total samples", tot)
    for k, v in sorted(lines.items(), key=lambda x: -x[1][2])[:n]:
        top = sorted(v[3].items(), key=lambda x: -x[1])[:3]
        print(f"{k[0][:8]:8s}{k[1]:5d} samp {100 * v[2] / max(tot, 1):5.1f}% inst {v[1]:9.0f} "
              f"{v[0].strip()[:58]:58s} {' '.join(f'{a}={b:.0f}' for a, b in top if b > 0)}")


if __name__ == "__main__":
    main()
