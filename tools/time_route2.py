"""Diagnostics (not a test): the refresh routing launch at the bench's C2
shape, route2_kernel vs route_fused_kernel (SPECSV_ROUTE_LEGACY), warm (one
cache) and cold (16 distinct caches, CUDA graph), CUDA events.

    python tools/time_route2.py [ctx] [gamma]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from tools.gpu_warm import spin_up  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cases = [build_case(ctx, g) for _ in range(16)]
    spin_up(0.5)
    for legacy in (False, True):
        if legacy:
            os.environ.pop("SPECSV_ROUTE2", None)
        else:
            os.environ["SPECSV_ROUTE2"] = "1"
        cfg, c, b, s, out, ws = cases[0]
        spin_up(0.2)
        warm = timed(lambda: V.route(cfg, c, b, s, out, ws))

        def all_cases():
            for cfg_, c_, b_, s_, o_, w_ in cases:
                V.route(cfg_, c_, b_, s_, o_, w_)

        all_cases()
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(gph, stream=st):
                all_cases()
        torch.cuda.current_stream().wait_stream(st)
        cold = timed(gph.replay, 10) / len(cases)
        print(f"{'legacy route_fused_kernel' if legacy else 'route2_kernel':26s} ctx={ctx} gamma={g}: "
              f"warm {warm:.1f} us, cold (graph over 16 caches) {cold:.1f} us per launch")


if __name__ == "__main__":
    main()
