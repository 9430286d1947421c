"""Diagnostics helper: keep the GPU busy long enough for its clocks to leave
the idle state before a short timing or trace run (a few microsecond-scale
launches after idle run at a fraction of the boost clock)."""
import time

import torch


def spin_up(seconds: float = 0.5) -> None:
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    t0 = time.time()
    while time.time() - t0 < seconds:
        for _ in range(20):
            a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()
