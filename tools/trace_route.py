"""Diagnostics (not a test): per-CTA phase timeline of one fused routing
launch at the bench shape (globaltimer stamps, us from the first CTA start).

    python tools/trace_route.py [ctx] [gamma]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from paper_2605_19893_b200 import abi  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402

BASE = 196608
NAMES = ["start", "tiles", "bar1", "shares", "bar2", "tail", "shares2", "tail2",
         "t:scores", "t:warpbest", "t:bound", "t:surv", "t:rank",
         "s:stats"]


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg, c, b, s, out, ws = build_case(ctx, g)
    for _ in range(3):
        V.route(cfg, c, b, s, out, ws)
    buf = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
    abi.lib().specsv_debug_attend_trace(buf.data_ptr())
    V.route(cfg, c, b, s, out, ws)
    torch.cuda.synchronize()
    abi.lib().specsv_debug_attend_trace(None)
    full = buf[BASE:BASE + 1024 * 64].view(-1, 64).cpu().numpy()
    for row in full[:9]:
        if row[15] > row[14] > 0 and row[5] > row[0]:
            print("tail CTA effective SM clock MHz:", (row[15] - row[14]) / ((row[5] - row[0]) / 1e3) / 1e6 * 1e3 / 1e3)
    t = full[:, :14]
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    print("ctas", len(t))
    names = ["prologue"] + [f"{n}{i}" for i in range(3) for n in ("mma", "store", "exp", "bar2", "gw")]
    for gname, off in (("grp0", 16), ("grp1", 32)):
        for k, name in enumerate(names):
            d = full[:len(t), off + k]
            d = (d[d > 0] - t0) / 1e3
            if len(d):
                print(f"{gname}.{name:9s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}")
    for k, name in enumerate(NAMES):
        d = t[:, k]
        d = (d[d > 0] - t0) / 1e3
        if len(d):
            print(f"{name:7s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}  (n={len(d)})")


if __name__ == "__main__":
    main()
