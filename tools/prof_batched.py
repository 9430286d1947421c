"""Diagnostics (not a test): a few batched verify calls at C4's shape (8
requests, 128K, gamma=8, exact C=4, all REFRESH) for ncu captures of
route_batch_kernel and nsa_attend_batch_kernel:

    ncu -k regex:route_batch --launch-skip 1 --launch-count 1 --set full -o out python tools/prof_batched.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402


def main():
    R, ctx, g = 8, 131072, 8
    nq = g + 1
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=1)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4)

    def urand(*shape, dtype=torch.float32):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(dtype)

    pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
    caches, batches, sets, outs = [], [], [], []
    for _ in range(R):
        c = V.LayerCache(cfg, ctx, device=dev)
        c.k.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
        c.v.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
        c.rows = ctx
        c.extend_compressed(urand(cfg.l, 128) * 0.1)
        caches.append(c)
        batches.append(V.DraftBatch(pos=pos, tree_mask=chain_tree_mask(g), q=urand(nq, 32, 128),
                                    gates=torch.rand(nq, 32, 3, generator=gen, device=dev),
                                    tree_k=urand(g, 8, 128, dtype=torch.bfloat16),
                                    tree_v=urand(g, 8, 128, dtype=torch.bfloat16)))
        sets.append(V.IndexSets.empty(nq, cfg.n, dev))
        outs.append(torch.zeros(nq, 32, 128, device=dev))
    ws = V.Workspace(cfg, nq, ctx, device=dev, batch=R)
    for _ in range(3):
        V.nsa_verify_batched(cfg, caches, batches, sets, outs, ws, 4, V.MODE_EXACT)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
