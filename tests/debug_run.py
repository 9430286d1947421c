"""Diagnostics for the GPU path (not a test): runs verify cases with one-hot
gates to isolate the compressed / selected / window branches, prints index
agreement and per-branch errors against the oracle.

    python tests/debug_run.py [rows] [gamma]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402
from tests.gpu_harness import DeviceCase, rel_errors, sets_to_numpy  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    gamma = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    lib = O.load("oracle")
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, rows, gamma, 7)
    t0 = time.time()
    case = DeviceCase(cfg, x)
    print("setup", time.time() - t0, "blocks", case.cache.blocks, flush=True)
    ck, cv = case.oracle_cache(lib)
    got_ck = case.cache.ck[:ck.shape[0]].cpu().numpy()
    print("ck bit-exact:", np.array_equal(got_ck.view(np.uint32), ck.view(np.uint32)), flush=True)
    sc = V.selection_scores(case.vcfg, case.cache, case.batch, 0, case.ws).cpu().numpy()
    rs = lib.selection_scores(cfg, x.q[0], ck, cfg.routing_visible_len(int(x.pos[0])))
    print("scores max rel diff:", float(np.abs(sc - rs).max() / np.abs(rs).max()), flush=True)
    for name, g in (("cmp", (1, 0, 0)), ("slc", (0, 1, 0)), ("win", (0, 0, 1)), ("all", None)):
        if g is not None:
            gates = np.zeros_like(x.gates)
            gates[..., :] = np.array(g, np.float32)
            case.batch.gates = torch.from_numpy(gates).cuda()
            x_g = gates
        else:
            case.batch.gates = torch.from_numpy(x.gates).cuda()
            x_g = x.gates
        out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
        saved = x.gates
        x.gates = x_g
        ref = case.oracle(lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
        x.gates = saved
        gi, gc, _ = sets_to_numpy(sets)
        same = [bool(gc[q] == ref["idx_count"][q] and (gi[q, :gc[q]] == ref["idx"][q, :gc[q]]).all())
                for q in range(1 + gamma)]
        per, l2 = rel_errors(out, ref["out"])
        print(f"{name}: idx_same={all(same)} per={per:.3e} l2={l2:.3e} "
              f"gpu[0,0,:4]={out[0, 0, :4]} ref={ref['out'][0, 0, :4]}", flush=True)
        if not all(same):
            print("  gpu idx q0", gi[0, :gc[0]], "\n  ref idx q0", ref["idx"][0, :ref["idx_count"][0]])
        bad = np.argwhere(np.abs(out - ref["out"]).max(-1) > 2e-3 * np.maximum(np.abs(ref["out"]).max(-1), 1e-6))
        if len(bad):
            print("  bad (q,h) first 10:", bad[:10].tolist())


if __name__ == "__main__" and len(sys.argv) <= 3:
    main()


def trace_attend(rows=65536, gamma=8):
    """Per-CTA phase timeline of one fused attend launch (globaltimer, ns)."""
    from paper_2605_19893_b200 import abi
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, rows, gamma, 9)
    case = DeviceCase(cfg, x)
    case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    buf = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
    abi.lib().specsv_debug_attend_trace(torch.cuda.LongTensor.data_ptr(buf))
    sets = V.IndexSets.empty(case.nq, cfg.n)
    out = torch.zeros(case.nq, cfg.n_q_heads, cfg.d_head, device="cuda")
    V.route(case.vcfg, case.cache, case.batch, sets, out, case.ws, 4)
    for _ in range(3):
        V.attend_fused(case.vcfg, case.cache, case.batch, sets, out, case.ws, 4, V.MODE_EXACT, V.ROLE_REUSE)
    torch.cuda.synchronize()
    abi.lib().specsv_debug_attend_trace(None)
    t = buf.view(-1, 64).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    for c in (0, 1, 17, 100):
        if c >= len(t):
            continue
        r = t[c]
        print(f"cta {c}: start {(r[0]-t0)/1e3:.2f} q_ready {(r[5]-t0)/1e3:.2f} setup {(r[1]-t0)/1e3:.2f} loop {(r[2]-t0)/1e3:.2f} "
              f"lastpv {(r[7]-t0)/1e3:.2f} part {(r[3]-t0)/1e3:.2f} barrier {(r[6]-t0)/1e3:.2f} merge {(r[4]-t0)/1e3:.2f}")
        print("   union: start %.2f staged %.2f prefix %.2f scatter %.2f done %.2f prefetched %.2f; q math %.2f" % tuple(
            (r[k] - t0) / 1e3 for k in (59, 56, 57, 58, 1, 60, 61)))
        for j in range(8):
            ev = [r[8 + j], r[16 + j], r[24 + j], r[56 + j], r[48 + j], r[32 + j], r[40 + j]]
            if ev[0] == 0:
                break
            print("   tile", j, " ".join(f"{(x - t0) / 1e3:7.2f}" if x else "   -   " for x in ev),
                  "(tma, qk, s_full, s_ld, vote, p_full, pv)")
    print("ctas", len(t), "fast-pass flags", np.unique(t[:, 62], return_counts=True),
          "robust-pass flags", np.unique(t[:, 63], return_counts=True))
    for name, col in (("setup", 1), ("tiles", 2), ("partials", 3), ("merge", 4)):
        d = (t[:, col] - t0) / 1e3
        print(f"{name:9s} done at us: min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}")
    print("start spread us:", (t[:, 0].max() - t0) / 1e3)


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "trace":
    trace_attend(int(sys.argv[1]), int(sys.argv[2]))
