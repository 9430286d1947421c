"""Diagnostics (not a test): where the bench's e2e step loses time against the
graph-replayed step.  C2 shape (64K, gamma 8, 32 layers, alt schedule):
device time (CUDA events) and host time per step for
  graph   : the captured step
  eager   : the 32 PreparedVerify calls, nothing else
  +commit : eager + the accepted-row commit and position update
  +copies : eager + the per-step pinned host->device input copies (copy stream)

    python tools/e2e_probe.py [steps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import tree as TR  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    L, ctx, g = 32, 65536, 8
    nq = g + 1
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=L)
    roles, source = V.resolve_layer_roles(list(range(1, L, 2)), L)
    cap = ctx + 2000
    torch.manual_seed(0)
    pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
    caches, batches, sets, outs = [], [], [], []
    pe = (torch.rand(cfg.l, 128, device=dev) * 2 - 1) * 0.1
    inbuf = torch.zeros(L, nq * 32 * 128 * 4, dtype=torch.uint8, device=dev)
    for j in range(L):
        c = V.LayerCache(cfg, cap, device=dev)
        c.k[:ctx].copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
        c.v[:ctx].copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
        c.rows = ctx
        c.extend_compressed(pe)
        caches.append(c)
        q = inbuf[j].view(torch.float32).view(nq, 32, 128)
        q.copy_(torch.rand(nq, 32, 128, device=dev) * 2 - 1)
        batches.append(V.DraftBatch(pos=pos.copy(), tree_mask=chain_tree_mask(g), q=q,
                                    gates=torch.rand(nq, 32, 3, device=dev) * 0.6 + 0.2,
                                    tree_k=(torch.rand(g, 8, 128, device=dev) * 2 - 1).bfloat16(),
                                    tree_v=(torch.rand(g, 8, 128, device=dev) * 2 - 1).bfloat16()))
        sets.append(V.IndexSets.empty(nq, cfg.n, dev))
        outs.append(torch.zeros(nq, 32, 128, device=dev))
    ws = V.Workspace(cfg, nq, cap, device=dev)
    prepared = [V.PreparedVerify(cfg, caches[j], batches[j], sets[j if roles[j] == V.ROLE_REFRESH else int(source[j])],
                                 outs[j], ws, 4, V.MODE_EXACT, int(roles[j])) for j in range(L)]
    commit = TR.PreparedCommit(cfg, caches, [b.tree_k for b in batches], [b.tree_v for b in batches],
                               [0, 1, 2, 3, 4], pe)
    hin = inbuf.cpu().pin_memory()
    cs = torch.cuda.Stream(device=dev)

    def eager(do_commit=False, do_copies=False):
        cur = torch.cuda.current_stream()
        if do_copies:
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                inbuf.copy_(hin, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            cur.wait_event(ev)
        for p in prepared:
            p.run()
        if do_commit:
            commit.run(cur)
            new_pos = np.array([caches[0].rows - 1 + i for i in range(nq)], np.int64)
            for b in batches:
                b.pos = new_pos

    def timed(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3, (t1 - t0) / n * 1e6

    # graph of the plain step
    gph = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        eager()
        torch.cuda.synchronize()
        with torch.cuda.graph(gph, stream=st):
            eager()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    for name, fn in [("graph", gph.replay), ("eager", eager), ("eager+commit", lambda: eager(True)),
                     ("eager+copies", lambda: eager(False, True)),
                     ("eager+commit+copies", lambda: eager(True, True))]:
        d, h = timed(fn, steps)
        print(f"{name:22s} device {d:8.1f} us/step   host {h:8.1f} us/step", flush=True)


if __name__ == "__main__":
    main()
