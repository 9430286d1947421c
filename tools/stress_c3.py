"""Diagnostics (not a test): repeat the C3 refresh layer (64K, 32-node tree,
exact C=4) on the GPU against ONE oracle result and report every run whose
per-(query, head) error exceeds the tolerance -- which (query, head, chunk)
and whether any attend CTA took the robust redo pass (trace flags).

    python tools/stress_c3.py [runs] [mode]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import abi  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402
from tests.gpu_harness import TOL, DeviceCase  # noqa: E402

TREE32 = [-1] * 4 + [i // 4 - 1 for i in range(4, 32)]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    runs = int(args[0]) if args else 40
    mode = int(args[1]) if len(args) > 1 else O.MODE_EXACT
    lib = O.load("oracle")
    cfg = O.llama_config(32)
    x = LayerInputs(cfg, 65536, 32, 3232, parent_slot=TREE32)
    br = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--branch=")), None)
    if br is not None:  # one-hot gates: the output is that branch alone
        x.gates = np.zeros_like(x.gates)
        x.gates[:, :, br] = 1.0
    case = DeviceCase(cfg, x)
    ref = case.oracle(lib, 4, mode, O.ROLE_REFRESH)["out"]
    den = np.maximum(np.abs(ref).max(axis=2), 1e-6)
    buf = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
    bad_runs = 0
    fresh = "--fresh" in sys.argv  # a new cache + workspace per run, no tracing (the test's setting)
    for it in range(runs):
        if fresh:
            case = DeviceCase(cfg, x)
            out, _ = case.run(4, mode, V.ROLE_REFRESH)
        else:
            abi.lib().specsv_debug_attend_trace(buf.data_ptr())
            buf.zero_()
            out, _ = case.run(4, mode, V.ROLE_REFRESH)
            abi.lib().specsv_debug_attend_trace(None)
        err = np.abs(out - ref).max(axis=2) / den
        t = buf.view(-1, 64).cpu().numpy()
        t = t[t[:, 0] > 0]
        robust = int((t[:, 62] != 0).sum())
        if err.max() > TOL:
            bad_runs += 1
            qs, hs = np.nonzero(err > TOL)
            print(f"run {it}: max err {err.max():.4f}; bad (q,h): "
                  f"{list(zip(qs.tolist(), hs.tolist()))[:12]} ({len(qs)} total); "
                  f"CTAs taking the robust pass: {robust}", flush=True)
        elif it % 10 == 0:
            print(f"run {it}: ok (max err {err.max():.2e}, robust CTAs {robust})", flush=True)
    print(f"{bad_runs} bad runs of {runs}")


if __name__ == "__main__":
    main()
