"""Diagnostics (not a test): per-CTA phase timeline of one route2 launch at
the bench shape (globaltimer stamps, us from the first CTA start).

    python tools/trace_route2.py [ctx] [gamma]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from paper_2605_19893_b200 import abi  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from tools.gpu_warm import spin_up  # noqa: E402

BASE = 196608
NAMES = {0: "start", 1: "tile 0 keys landed", 11: "warp 0: tile 0 DMMA done",
         14: "warp 8: tile 0 epilogue done", 12: "warp 0: all its DMMA done", 2: "tiles done",
         10: "fold max/den", 3: "fold done", 4: "barrier passed", 5: "shares written",
         6: "range scores (last writers)", 7: "candidates", 8: "final gather", 9: "final merge"}
GHZ = 1.965  # stamps are SM cycles since each CTA's start


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cases = [build_case(ctx, g) for _ in range(2)]
    for c in cases:
        V.route(*c)
    buf = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
    for trial in range(2):
        buf.zero_()
        cfg, c, b, s, out, ws = cases[trial]
        spin_up(0.3)
        for _ in range(200):  # back-to-back launches right before the traced one
            V.route(cfg, c, b, s, out, ws)
        abi.lib().specsv_debug_attend_trace(buf.data_ptr())
        V.route(cfg, c, b, s, out, ws)
        torch.cuda.synchronize()
        abi.lib().specsv_debug_attend_trace(None)
        t = buf[BASE:BASE + 1024 * 16].view(-1, 16).cpu().numpy()
        t = t[t[:, 0] > 0]
        print(f"trial {trial}: ctas {len(t)}  (us from each CTA's start, SM cycles / {GHZ} GHz)")
        for k, name in NAMES.items():
            d = t[:, k]
            d = d[d > 0] / GHZ / 1e3
            if len(d):
                print(f"  {name:30s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}  (n={len(d)})")


if __name__ == "__main__":
    main()
