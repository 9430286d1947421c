"""Diagnostics (not a test): routing cost per request at C4's shape (128K,
gamma=8, exact C=4) -- single routing launches against one batched routing
launch (nsa_verify_batched REFRESH minus REUSE), graph-timed.

    python tools/time_batched.py [R] [ctx]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402
from tools.sweep import graph_time  # noqa: E402


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=1)
    g, nq = 8, 9
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)

    def urand(*shape, dtype=torch.float32):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(dtype)

    caches, batches, sets, outs = [], [], [], []
    pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
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
    ws = V.Workspace(cfg, nq, ctx, device=dev, batch=min(R, 16))
    single_route = graph_time(lambda: [V.route(cfg, caches[r], batches[r], sets[r], outs[r], ws)
                                       for r in range(R)])
    single_att = graph_time(lambda: [V.attend_fused(cfg, caches[r], batches[r], sets[r], outs[r], ws, 4,
                                                    V.MODE_EXACT, V.ROLE_REUSE) for r in range(R)])
    b_ref = graph_time(lambda: V.nsa_verify_batched(cfg, caches, batches, sets, outs, ws, 4, V.MODE_EXACT,
                                                    [V.ROLE_REFRESH] * R))
    b_reu = graph_time(lambda: V.nsa_verify_batched(cfg, caches, batches, sets, outs, ws, 4, V.MODE_EXACT,
                                                    [V.ROLE_REUSE] * R))
    print(f"R={R} ctx={ctx}: per request  single route {single_route / R * 1e3:.1f} us, "
          f"single attend {single_att / R * 1e3:.1f} us | batched attend {b_reu / R * 1e3:.1f} us, "
          f"batched routing {(b_ref - b_reu) / R * 1e3:.1f} us")


if __name__ == "__main__":
    main()
