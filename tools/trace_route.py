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
NAMES = {32: "item0 stage", 33: "item0 staged", 48: "item0 mma done", 49: "item1 mma done", 34: "item0 computed", 35: "item1 stage",
         36: "item1 staged", 37: "item1 computed", 0: "start", 1: "tiles done", 4: "barrier passed", 13: "unit staged", 7: "F written", 14: "part written", 8: "slot atomic", 15: "sel summed",
         9: "topn warp-best", 10: "topn bound", 11: "topn survivors", 12: "topn rank", 5: "tail done"}


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
    t = buf[BASE:BASE + 1024 * 64].view(-1, 64).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    print("ctas", len(t))
    for k, name in NAMES.items():
        d = t[:, k]
        d = (d[d > 0] - t0) / 1e3
        if len(d):
            print(f"{name:16s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}  (n={len(d)})")


if __name__ == "__main__":
    main()
