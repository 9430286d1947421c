"""Diagnostics (not a test): times the refresh-layer routing launch chain
(R1 logits, R2 mass, R3 Top-n) at the bench's 64K / gamma=8 / exact shape
with CUDA events.  SPECSV_ROUTE_DEBUG=<bits> skips R1 phases (1: MMA loop,
2: exp, 4: fold, 8: E stores) -- parity is void under it.

    python tools/time_route.py [ctx] [gamma]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402


def build_case(ctx, g):
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=1, n_q_heads=32, n_kv_heads=8, d_head=128)
    nq = g + 1
    torch.manual_seed(0)
    c = V.LayerCache(cfg, ctx, device=dev)
    c.k.copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
    c.v.copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
    c.rows = ctx
    c.extend_compressed((torch.rand(cfg.l, 128, device=dev) * 2 - 1) * 0.1)
    pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
    b = V.DraftBatch(pos=pos, tree_mask=chain_tree_mask(g),
                     q=torch.rand(nq, 32, 128, device=dev) * 2 - 1,
                     gates=torch.rand(nq, 32, 3, device=dev),
                     tree_k=torch.rand(g, 8, 128, device=dev).bfloat16(),
                     tree_v=torch.rand(g, 8, 128, device=dev).bfloat16())
    s = V.IndexSets.empty(nq, cfg.n, dev)
    out = torch.zeros(nq, 32, 128, device=dev)
    ws = V.Workspace(cfg, nq, ctx, device=dev)
    return cfg, c, b, s, out, ws


def main():
    ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg, c, b, s, out, ws = build_case(ctx, g)
    for _ in range(5):
        V.route(cfg, c, b, s, out, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 50
    for _ in range(n):
        V.route(cfg, c, b, s, out, ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"route ctx={ctx} gamma={g} flags={os.environ.get('SPECSV_ROUTE_DEBUG', '0')}: "
          f"{e0.elapsed_time(e1) / n * 1000:.1f} us per launch chain")


if __name__ == "__main__":
    main()
