"""Diagnostics (not a test): the refresh routing launch at the bench's C2
shape -- route3_kernel (default) vs route_fused_kernel (SPECSV_ROUTE_LEGACY=1)
-- warm (one cache) and cold (16 distinct caches, CUDA graph), CUDA events;
plus route3's exact re-scoring count and per-phase stamps.

    python tools/time_route3.py [ctx] [gamma]

The per-phase stamps need the diagnostics build
(SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force);
the default build prints the launch timings only.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from tools.gpu_warm import spin_up  # noqa: E402
from paper_2605_19893_b200 import abi  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402

BASE = 196608
PHASES = {1: "q digits staged", 9: "tile 0 MMAs done", 10: "tile 1 MMAs done", 2: "e values done",
          3: "unit sums done", 4: "phase 1 done",
          5: "den rows in", 6: "shares written", 7: "top-n start", 14: "top-n scores in", 15: "top-n selected",
          8: "done"}


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
            os.environ["SPECSV_ROUTE_LEGACY"] = "1"
        else:
            os.environ.pop("SPECSV_ROUTE_LEGACY", None)
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
        name = "legacy route_fused_kernel" if legacy else "route3_kernel"
        print(f"{name:26s} ctx={ctx} gamma={g}: warm {warm:.1f} us, cold (graph over 16 caches) "
              f"{cold:.1f} us per launch", flush=True)
    os.environ.pop("SPECSV_ROUTE_LEGACY", None)
    # phase stamps of one cold launch
    cfg, c, b, s, out, ws = cases[3]
    buf = torch.zeros(BASE + 4096 * 16, dtype=torch.int64, device="cuda")
    for _ in range(50):
        V.route(*cases[(_ % 15) + 1])
    abi.lib().specsv_debug_attend_trace(buf.data_ptr())
    V.route(cfg, c, b, s, out, ws)
    torch.cuda.synchronize()
    abi.lib().specsv_debug_attend_trace(None)
    t = buf[BASE:].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    print(f"route3 phases ({len(t)} CTAs, us from the first CTA start):")
    for k, name in PHASES.items():
        d = t[:, k]
        d = d[d > 0]
        if len(d):
            d = (d - t0) / 1e3
            print(f"  {name:22s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}  (n={len(d)})")
    tk = t[t[:, 12] > 0]
    if len(tk):
        print(f"  select: {np.median(tk[:, 12]):.0f} SM cycles (median over {len(tk)} tasks), "
              f"of which steps 1-2 {np.median(tk[:, 11]):.0f}")
    d = (t[:, 0] - t0) / 1e3
    print(f"  {'start':22s} min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}")
    print("exact re-scorings:", sum(cs[-1].route_fallbacks() for cs in cases), "over all launches")


if __name__ == "__main__":
    main()
