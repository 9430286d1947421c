"""Diagnostics (not a test): device fp64 selection scores vs the oracle for one case."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402
from tests.gpu_harness import DeviceCase  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3001
gamma = int(sys.argv[2]) if len(sys.argv) > 2 else 8
parents = [-1, -1, 0, 0, 1, 2, 2, 4] if gamma == 8 else None
lib = O.load("oracle")
cfg = O.llama_config(4)
x = LayerInputs(cfg, rows, gamma, 100 + rows + gamma, parent_slot=parents)
case = DeviceCase(cfg, x)
ck, _ = case.oracle_cache(lib)
for q in range(case.nq):
    got = V.selection_scores(case.vcfg, case.cache, case.batch, q, case.ws).cpu().numpy()
    ref = lib.selection_scores(cfg, x.q[q], ck, cfg.routing_visible_len(int(x.pos[q])))
    d = np.abs(got - ref) / np.abs(ref).max()
    print(q, got.shape, ref.shape, "max rel", d.max(), "at", int(d.argmax()), got[d.argmax()], ref[d.argmax()])
