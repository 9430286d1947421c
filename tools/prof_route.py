"""Diagnostics (not a test): routing launches at the bench's C2 shape for ncu
captures of the route kernel:

    ncu -k regex:route_fused --launch-skip 2 --launch-count 1 --set full \
        --import-source on -o gpurun_out/route python tools/prof_route.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.time_route import build_case  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402


def main():
    cfg, c, b, s, out, ws = build_case(65536, 8)
    for _ in range(4):
        V.route(cfg, c, b, s, out, ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
