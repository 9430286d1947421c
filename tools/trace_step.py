"""Diagnostics (not a test): per-kernel phase timeline of the bench step in
its real setting -- distinct 64K layer caches (cold L2), one CUDA graph of
`L` verify calls ("alt" refresh/reuse) -- from the kernels' globaltimer
stamps (specsv_debug_attend_trace; one trace buffer per layer).

    python tools/trace_step.py [layers] [ctx] [gamma]

Per-tile columns (TRACE_TILES=1), the routing phases and the union / producer
stamps need the diagnostics build (SPECSV_TRACE_TILES=1 python -m
paper_2605_19893_b200.build --force); the per-CTA attend phases are in every
build.

Prints, per layer, the attend kernel's first-CTA start, the median/max CTA
phase times (union built, tile loop done, partials written, barrier passed,
merge done, relative to the first CTA start) and the gap to the previous
kernel's last CTA end; refresh layers also show the routing kernel.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19893_b200 import abi  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import chain_tree_mask  # noqa: E402

RBASE = 196608


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    g = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    dev = torch.device("cuda", 0)
    cfg = V.NsaConfig(n_layers=L)
    nq = g + 1
    torch.manual_seed(0)
    pos = np.array([ctx - 1 + i for i in range(nq)], np.int64)
    layers = []
    for j in range(L):
        c = V.LayerCache(cfg, ctx, device=dev)
        c.k.copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
        c.v.copy_((torch.rand(ctx, 8, 128, device=dev) * 2 - 1).bfloat16())
        c.rows = ctx
        c.extend_compressed((torch.rand(cfg.l, 128, device=dev) * 2 - 1) * 0.1)
        b = V.DraftBatch(pos=pos, tree_mask=chain_tree_mask(g),
                         q=torch.rand(nq, 32, 128, device=dev) * 2 - 1,
                         gates=torch.rand(nq, 32, 3, device=dev) * 0.6 + 0.2,
                         tree_k=(torch.rand(g, 8, 128, device=dev) * 2 - 1).bfloat16(),
                         tree_v=(torch.rand(g, 8, 128, device=dev) * 2 - 1).bfloat16())
        layers.append((c, b, V.IndexSets.empty(nq, cfg.n, dev), torch.zeros(nq, 32, 128, device=dev)))
    ws = V.Workspace(cfg, nq, ctx, device=dev)
    bufs = [torch.zeros(4096 * 64, dtype=torch.int64, device=dev) for _ in range(L)]

    def step(trace):
        for j in range(L):
            if trace:
                abi.lib().specsv_debug_attend_trace(bufs[j].data_ptr())
            c, b, s, o = layers[j]
            refresh = j % 2 == 0
            src = s if refresh else layers[j - 1][2]
            V.nsa_verify(cfg, c, b, src, o, ws, 4, V.MODE_EXACT,
                         V.ROLE_REFRESH if refresh else V.ROLE_REUSE)
        abi.lib().specsv_debug_attend_trace(None)

    step(False)
    torch.cuda.synchronize()
    if os.environ.get("TRACE_EAGER"):  # the same calls issued eagerly (no graph)
        for _ in range(3):
            step(False)
        torch.cuda.synchronize()
        for bb in bufs:
            bb.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step(True)
        e1.record()
        torch.cuda.synchronize()
        print(f"step of {L} layers: {e0.elapsed_time(e1) * 1e3:.1f} us (traced, eager)")
        report(L, bufs)
        return
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            step(True)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for bb in bufs:
        bb.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"step of {L} layers: {e0.elapsed_time(e1) * 1e3:.1f} us (traced)")
    report(L, bufs)


def report(L, bufs):
    t_first = None
    prev_end = None
    for j in range(L):
        t = bufs[j][:RBASE].view(-1, 64).cpu().numpy()
        t = t[t[:, 0] > 0]
        r = bufs[j][RBASE:RBASE + 1024 * 16].view(-1, 16).cpu().numpy()
        r = r[r[:, 0] > 0]
        if t_first is None:
            t_first = (r[:, 0].min() if len(r) else t[:, 0].min())
        line = f"layer {j:2d} {'R' if j % 2 == 0 else 'U'}"
        if len(r):  # route3 stamps: 0 start, 4 phase 1 done, 6 shares written, 8 done
            r0 = r[:, 0].min()
            rend = r[:, 8].max()
            gap = (r0 - prev_end) / 1e3 if prev_end is not None else 0.0
            p1 = (np.median(r[:, 4][r[:, 4] > 0]) - r0) / 1e3
            sh = (np.median(r[:, 6][r[:, 6] > 0]) - r0) / 1e3
            tk = r[r[:, 7] > 0]  # the Top-n task CTAs: start, scores in, selected, done

            def tcol(c):
                return (np.median(tk[:, c]) - r0) / 1e3 if len(tk) else -1
            line += (f" | route start {(r0 - t_first) / 1e3:8.2f} gap {gap:5.2f} phase1(med) {p1:5.2f}"
                     f" shares {sh:5.2f} topn {tcol(7):5.2f}/{tcol(14):5.2f}/{tcol(15):5.2f}/{tcol(8):5.2f}"
                     f" select {np.median(tk[:, 12]) if len(tk) else -1:.0f} clk"
                     f" end {(rend - r0) / 1e3:5.2f}")
            prev_end = rend
        t0 = t[:, 0].min()
        gap = (t0 - prev_end) / 1e3 if prev_end is not None else 0.0

        def ph(col):
            d = t[:, col]
            d = d[d > 0]
            return ((np.median(d) - t0) / 1e3, (d.max() - t0) / 1e3) if len(d) else (-1, -1)

        end = t[:, 4].max()
        line += (f" | attend start {(t0 - t_first) / 1e3:8.2f} gap {gap:5.2f} spread {(t[:, 0].max() - t0) / 1e3:4.2f}"
                 f" idx in {ph(59)[0]:5.2f}/{ph(59)[1]:5.2f}"
                 f" union {ph(1)[0]:5.2f} loop {ph(2)[0]:5.2f}/{ph(2)[1]:5.2f} pv {ph(7)[0]:5.2f}/{ph(7)[1]:5.2f} part {ph(3)[0]:5.2f}/{ph(3)[1]:5.2f}"
                 f" bar {ph(6)[0]:5.2f} merge {ph(4)[0]:5.2f}/{ph(4)[1]:5.2f} ctas {len(t)}")
        prev_end = end
        print(line)
        if os.environ.get("TRACE_HEADS"):  # per KV head (CTA id = head * 18 + split)
            full = bufs[j][:RBASE].view(-1, 64).cpu().numpy()[:144]
            for h in range(8):
                hb = full[h * 18:(h + 1) * 18]
                st, le = (hb[:, 0] - t0) / 1e3, (hb[:, 2] - t0) / 1e3
                print(f"   head {h}: start {st.min():5.2f}-{st.max():5.2f} loop end med {np.median(le):5.2f} "
                      f"max {le.max():5.2f} (split {int(le.argmax())}) merge {((hb[:, 4] - t0) / 1e3).max():5.2f}")
        if os.environ.get("TRACE_TILES"):
            print_tiles(t)
        if os.environ.get("TRACE_SPLITS"):
            print("   split: loop end / partials written (median over heads): " +
                  " ".join(f"{sp}:{a:.1f}/{b:.1f}" for sp, a, b in per_split(bufs[j])))


def print_tiles(t):
    """per-tile stamps (median over CTAs, us from each CTA's own start):
    TMA issue, K full (QK issued), S full (softmax start), exp done, P handed
    over, V full (PV issued)"""
    raw = t[:, [0, 16, 24, 48, 32, 40]].astype(np.int64).ravel()
    raw = raw[raw > 0]
    print("   globaltimer gcd of stamps (ns):", int(np.gcd.reduce(raw - raw.min())),
          " distinct low values:", len(np.unique(raw % 1000)))
    rel = (t - t[:, :1]) / 1e3
    cols = [("issue", 8), ("qk", 16), ("s_full", 24), ("exp", 48), ("p", 32), ("pv", 40)]
    u = [np.median(rel[:, c][t[:, c] > 0]) if (t[:, c] > 0).sum() > len(t) // 2 else -1
         for c in (59, 56, 57, 58, 60, 1)]
    chk = t[:, 63]
    if (chk >= 1000).any():
        print("   union check: %d CTAs checked, %d bad (codes %s)" % ((chk >= 1000).sum(), (chk > 1000).sum(),
                                                                  sorted(set((chk[chk > 1000] - 1000).tolist()))))
    print("   union: index rows in %.2f, built %.2f (us)" % (u[0], u[5]))
    if (t[:, 57] > 0).sum() > len(t) // 2:
        print("   producer: K2 %.2f-%.2f, V2 %.2f-%.2f, K3 %.2f-%.2f" %
              tuple(np.median(rel[:, c][t[:, c] > 0]) for c in (10, 56, 57, 58, 11, 60)))
    if os.environ.get("TRACE_RAW"):
        for i in range(0, len(t), 29):
            print("   cta %3d: " % i + " ".join("%d:%.2f" % (c, rel[i, c]) for c in (59, 56, 1, 24, 25, 26)))
    cyc = [int(np.median(t[:, c][t[:, c] > 0])) if (t[:, c] > 0).sum() > len(t) // 4 else -1
           for c in (29, 30, 31, 37, 38, 39, 47)]
    print("   softmax tile 3 (SM cycles from loop top): masks %d, S in %d, S read %d, exp %d, P free %d, "
          "P written %d, handed over %d" % tuple(cyc))
    print("   tile " + " ".join(f"{n:>8s}" for n, _ in cols))
    for j in range(8):
        vals = []
        for _, b in cols:
            d = rel[:, b + j][t[:, b + j] > 0]
            vals.append(f"{np.median(d):8.2f}" if len(d) > len(t) // 2 else "       -")
        print(f"   {j:4d} " + " ".join(vals))


def per_split(buf, S=18):
    """loop-end time per split index (median over KV heads) of one attend trace buffer"""
    t = buf[:RBASE].view(-1, 64).cpu().numpy()
    n = (t[:, 0] > 0).sum()
    t = t[:n]
    t0 = t[:, 0].min()
    rows = []
    for s in range(S):
        sel = t[s::S]
        rows.append((s, np.median((sel[:, 2] - t0) / 1e3), np.median((sel[:, 3] - t0) / 1e3)))
    return rows


if __name__ == "__main__":
    main()

