"""BASELINE configs C3 and C5 on one B200 (measurement tool, not a test).

C5: draft length gamma in {2, 4, 8, 16} x reuse fraction in {0, 0.5, 0.75}
    x context in {16K, 32K, 64K, 128K}: the verify step (L layer caches, a
    CUDA graph of nsa_verify calls) against per-query NSA decode on the same
    GPU and caches (the 1 + gamma queries as sequential single-query refresh
    calls, C = 1) -- the north star's ">= 3x" comparison.
C3: a 32-node draft tree at 64K context with the alt refresh/reuse schedule,
    exact and approx (C = 4).

Synthetic U[-1,1] KV / queries (no checkpoint).  Writes one JSON record per
configuration plus a summary:  python tools/sweep.py [out.json] [--quick]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import (chain_tree_mask, depths_from_parents,  # noqa: E402
                                            tree_mask_from_parents)

L = 8
REUSE = {0.0: [], 0.5: [1, 3, 5, 7], 0.75: [1, 2, 3, 5, 6, 7]}
TREE32 = [-1] * 4 + [i // 4 - 1 for i in range(4, 32)]


def graph_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps  # ms


def main():
    out_path = next((a for a in sys.argv[1:] if not a.startswith("--")), "gpurun_out/sweep.json")
    quick = "--quick" in sys.argv
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=L)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)

    def urand(*shape, dtype=torch.float32):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(dtype)

    records = []
    contexts = (16384, 65536) if quick else (16384, 32768, 65536, 131072)
    for ctx in contexts:
        caches = []
        for _ in range(L):
            c = V.LayerCache(cfg, ctx, device=dev)
            c.k.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
            c.v.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
            c.rows = ctx
            c.extend_compressed(urand(cfg.l, 128) * 0.1)
            caches.append(c)
        drafts = [("chain", g, None) for g in ((2, 8) if quick else (2, 4, 8, 16))]
        if ctx == 65536:
            drafts.append(("tree32", 32, TREE32))
        for kind, gamma, parents in drafts:
            nq = gamma + 1
            if parents is None:
                pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
                tmask = chain_tree_mask(gamma)
            else:
                pos = np.array([ctx - 1] + [ctx - 1 + d for d in depths_from_parents(parents)], np.int64)
                tmask = tree_mask_from_parents(parents)
            batches = [V.DraftBatch(pos=pos, tree_mask=tmask, q=urand(nq, 32, 128),
                                    gates=torch.rand(nq, 32, 3, generator=gen, device=dev) * 0.6 + 0.2,
                                    tree_k=urand(gamma, 8, 128, dtype=torch.bfloat16),
                                    tree_v=urand(gamma, 8, 128, dtype=torch.bfloat16)) for _ in range(L)]
            ws = V.Workspace(cfg, nq, ctx, device=dev)
            outs = [torch.zeros(nq, 32, 128, device=dev) for _ in range(L)]
            # per-query decode of the same 1 + gamma queries (C = 1, refresh every layer)
            ws1 = V.Workspace(cfg, 1, ctx, device=dev)
            dec = [(j, V.DraftBatch(pos=np.array([ctx - 1], np.int64), tree_mask=chain_tree_mask(0),
                                    q=batches[j].q[i:i + 1], gates=batches[j].gates[i:i + 1],
                                    tree_k=None, tree_v=None),
                    V.IndexSets.empty(1, cfg.n, dev), torch.zeros(1, 32, 128, device=dev))
                   for j in range(L) for i in range(nq)]

            def decode():
                for j, b1, s1, o1 in dec:
                    V.nsa_verify(cfg, caches[j], b1, s1, o1, ws1, 1, V.MODE_EXACT, V.ROLE_REFRESH)

            dec_ms = graph_time(decode, reps=3)
            fracs = (0.0, 0.5) if (quick or kind == "tree32") else (0.0, 0.5, 0.75)
            modes = ((V.MODE_EXACT, 4), (V.MODE_APPROX, 4)) if kind == "tree32" else ((V.MODE_EXACT, 4),)
            for frac in fracs:
                S = REUSE[frac]
                roles, source = V.resolve_layer_roles(S, L)
                for mode, C_ in modes:
                    sets = [V.IndexSets.empty(nq, cfg.n, dev) for _ in range(L)]

                    def step():
                        for j in range(L):
                            s = sets[j] if roles[j] == V.ROLE_REFRESH else sets[int(source[j])]
                            V.nsa_verify(cfg, caches[j], batches[j], s, outs[j], ws, C_, mode,
                                         int(roles[j]))

                    ms = graph_time(step)
                    rec = {"config": "C3" if kind == "tree32" else "C5", "draft": kind, "ctx": ctx,
                           "gamma": gamma, "reuse_fraction": frac, "layers": L,
                           "mode": "exact" if mode == V.MODE_EXACT else "approx", "C": C_,
                           "verify_ms_per_step": ms, "verify_qtok_s": nq / (ms * 1e-3),
                           "decode_ms_per_step": dec_ms, "decode_qtok_s": nq / (dec_ms * 1e-3),
                           "verify_speedup_vs_decode": dec_ms / ms}
                    records.append(rec)
                    print(json.dumps(rec), flush=True)
        del caches
        torch.cuda.empty_cache()
    sp = [r["verify_speedup_vs_decode"] for r in records]
    res = {"what": "BASELINE C3 / C5 on one B200: verify step vs per-query NSA decode, "
                   f"{L} layer caches per step, synthetic data",
           "gpu": torch.cuda.get_device_name(0),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "speedup_min": min(sp), "speedup_median": float(np.median(sp)), "speedup_max": max(sp),
           "records": records}
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "records"}, indent=1))


if __name__ == "__main__":
    main()
