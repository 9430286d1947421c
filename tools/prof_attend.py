"""Diagnostics (not a test): one routing launch plus a few fused attend
launches at the bench's C2 shape (64K ctx, 8-token chain, exact C=4), for
ncu captures of the attend kernel:

    ncu -k regex:nsa_attend --launch-skip 2 --launch-count 1 --set full \
        --import-source on -o gpurun_out/attend python tools/prof_attend.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg, c, b, s, out, ws = build_case(ctx, g)
    V.route(cfg, c, b, s, out, ws)
    for _ in range(4):
        V.attend_fused(cfg, c, b, s, out, ws, 4, V.MODE_EXACT, V.ROLE_REUSE)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        V.attend_fused(cfg, c, b, s, out, ws, 4, V.MODE_EXACT, V.ROLE_REUSE)
    e1.record()
    torch.cuda.synchronize()
    print(f"attend (same cache, L2-warm) {e0.elapsed_time(e1) / 20 * 1000:.1f} us per launch")


if __name__ == "__main__":
    main()
