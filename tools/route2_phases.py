"""Diagnostics (not a test): route2_kernel timed with CUDA events when it
returns early after phase k (SPECSV_ROUTE2_DEBUG_EXIT=k; results are void),
so successive differences give each phase's cost at full clocks.

    python tools/route2_phases.py [ctx] [gamma]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from tools.time_route2 import timed  # noqa: E402
from tools.gpu_warm import spin_up  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402

NAMES = {9: "launch only (empty kernel)", 1: "prologue + tiles", 2: "+ fold", 3: "+ range barrier", 4: "+ den, shares, range arrivals",
         5: "+ range scores, candidates", 0: "full (+ final merge)"}


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg, c, b, s, out, ws = build_case(ctx, g)
    os.environ["SPECSV_ROUTE2"] = "1"
    spin_up(0.5)
    # graph-replayed (no host work between launches)
    for k in (9, 1, 2, 3, 4, 5, 0):
        os.environ["SPECSV_ROUTE2_DEBUG_EXIT"] = str(k)
        V.route(cfg, c, b, s, out, ws)
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(gph, stream=st):
                for _ in range(20):
                    V.route(cfg, c, b, s, out, ws)
        torch.cuda.current_stream().wait_stream(st)
        us = timed(gph.replay, 10) / 20
        print(f"graph, exit after {k}: {us:7.1f} us  ({NAMES[k]})", flush=True)
    os.environ.pop("SPECSV_ROUTE2_DEBUG_EXIT")
    os.environ.pop("SPECSV_ROUTE2", None)
    print(f"legacy eager: {timed(lambda: V.route(cfg, c, b, s, out, ws), 50):7.1f} us")


if __name__ == "__main__":
    main()
