"""Calibrate the planner's linear step-latency model (planner.h cost model,
cost_model.cpp:78-131 semantics) to verify steps measured on this GPU.

For a grid of (context, draft length, group size C, mode, reuse schedule)
it times one verify step over L layer caches (a CUDA graph of nsa_verify
calls, CUDA events), derives the step accounting from the LoadStats of the
index sets the step actually used (specsv_load_stats + account_step) and
fits the coefficients by nonnegative least squares.  Writes the samples and
the fit as JSON (the planner's cost model "fed by GPU-measured LoadStats").

    python tools/calibrate_cost.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import planner as P  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402

L = 8


def schedule(name):
    return [] if name == "none" else list(range(1, L, 2))


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cost_fit.json"
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=L)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)

    def urand(*shape, dtype=torch.float32):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(dtype)

    samples, rows_out = [], []
    for ctx in (16384, 65536):
        caches = []
        for _ in range(L):
            c = V.LayerCache(cfg, ctx, device=dev)
            c.k.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
            c.v.copy_(urand(ctx, 8, 128, dtype=torch.bfloat16))
            c.rows = ctx
            c.extend_compressed(urand(cfg.l, 128) * 0.1)
            caches.append(c)
        for gamma in (4, 8, 16):
            nq = gamma + 1
            pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
            tmask = chain_tree_mask(gamma)
            batches = [V.DraftBatch(pos=pos, tree_mask=tmask, q=urand(nq, 32, 128),
                                    gates=torch.rand(nq, 32, 3, generator=gen, device=dev) * 0.6 + 0.2,
                                    tree_k=urand(gamma, 8, 128, dtype=torch.bfloat16),
                                    tree_v=urand(gamma, 8, 128, dtype=torch.bfloat16))
                       for _ in range(L)]
            ws = V.Workspace(cfg, nq, ctx, device=dev)
            outs = [torch.zeros(nq, 32, 128, device=dev) for _ in range(L)]
            for C_ in (1, 4):
                for mode in (V.MODE_EXACT, V.MODE_APPROX):
                    for sname in ("none", "alt"):
                        S = schedule(sname)
                        roles, source = V.resolve_layer_roles(S, L)
                        sets = [V.IndexSets.empty(nq, cfg.n, dev) for _ in range(L)]

                        def step():
                            for j in range(L):
                                s = sets[j] if roles[j] == V.ROLE_REFRESH else sets[int(source[j])]
                                V.nsa_verify(cfg, caches[j], batches[j], s, outs[j], ws, C_, mode,
                                             int(roles[j]))

                        step()
                        torch.cuda.synchronize()
                        g = torch.cuda.CUDAGraph()
                        st = torch.cuda.Stream()
                        st.wait_stream(torch.cuda.current_stream())
                        with torch.cuda.stream(st):
                            with torch.cuda.graph(g, stream=st):
                                step()
                        torch.cuda.current_stream().wait_stream(st)
                        for _ in range(3):
                            g.replay()
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        for _ in range(10):
                            g.replay()
                        e1.record()
                        torch.cuda.synchronize()
                        us = e0.elapsed_time(e1) / 10 * 1e3
                        per_layer = []
                        for j in range(L):
                            s = sets[j] if roles[j] == V.ROLE_REFRESH else sets[int(source[j])]
                            per_layer.append(V.load_stats(cfg, ctx, pos, tmask, s.idx.cpu().numpy(),
                                                          s.count.cpu().numpy(), C_, mode,
                                                          int(roles[j])))
                        acc = P.account_step(per_layer, S, L)
                        samples.append((acc, us))
                        rows_out.append({"ctx": ctx, "gamma": gamma, "C": C_,
                                         "mode": "exact" if mode == V.MODE_EXACT else "approx",
                                         "schedule": sname, "step_us": us,
                                         "accounting": acc.__dict__})
                        print(f"ctx={ctx} gamma={gamma} C={C_} mode={mode} S={sname}: {us:8.1f} us "
                              f"{acc}", flush=True)
        del caches
        torch.cuda.empty_cache()
    fit = P.fit_cost_coeffs(samples)
    pred = [P.estimate_latency(a, fit) for a, _ in samples]
    meas = [t for _, t in samples]
    rel = [abs(p - m) / m for p, m in zip(pred, meas)]
    res = {"what": "planner cost model (cost_model.cpp) fitted to measured verify steps, "
                   f"{L} layers per step, microseconds",
           "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "coeffs_us": fit.__dict__, "median_rel_error": float(np.median(rel)),
           "max_rel_error": float(np.max(rel)), "samples": rows_out}
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "samples"}, indent=1))


if __name__ == "__main__":
    main()
