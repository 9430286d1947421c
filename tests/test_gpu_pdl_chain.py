"""Back-to-back verify calls under programmatic dependent launch.

The attend launch triggers its dependents after its tile loop, before its
split merge and output writes, and every launch waits for its predecessor
before it writes the shared workspace (nsa_verify.h, "Programmatic dependent
launch").  A race there would show up when calls follow each other on one
stream with one workspace and no host synchronisation, as in the engine's
per-layer loop (engine.cpp:175-278: route on refresh layers, attend on every
layer).  Each call of such a chain must give exactly (bit for bit) what the
same call gives when it runs alone: same launch configuration, so the same
fp32 summation order.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402
from tests.gpu_harness import DeviceCase, sets_to_numpy  # noqa: E402

pytestmark = pytest.mark.gpu

ROWS, GAMMA, LAYERS, ROUNDS = 20000, 8, 6, 3


def _sequence():
    """refresh, reuse, refresh, reuse, ... (the `alt` schedule)"""
    return [V.ROLE_REFRESH if j % 2 == 0 else V.ROLE_REUSE for j in range(LAYERS)]


def _run(cases, ws, sets, outs, roles, sync_each):
    for j, case in enumerate(cases):
        src = j if roles[j] == V.ROLE_REFRESH else j - 1
        V.nsa_verify(case.vcfg, case.cache, case.batch, sets[src], outs[j], ws, 4, V.MODE_EXACT,
                     roles[j])
        if sync_each:
            torch.cuda.synchronize()


def test_back_to_back_calls_equal_isolated_calls():
    cfg = O.llama_config(LAYERS)
    cases = [DeviceCase(cfg, LayerInputs(cfg, ROWS, GAMMA, 7100 + j)) for j in range(LAYERS)]
    ws = cases[0].ws  # one workspace for the whole chain, as in a real step
    roles = _sequence()
    nq = cases[0].nq

    def fresh():
        sets = [V.IndexSets.empty(nq, cfg.n) for _ in range(LAYERS)]
        outs = [torch.full((nq, cfg.n_q_heads, cfg.d_head), float("nan"), device="cuda")
                for _ in range(LAYERS)]
        return sets, outs

    ref_sets, ref_outs = fresh()
    _run(cases, ws, ref_sets, ref_outs, roles, sync_each=True)
    ref = [o.cpu().numpy() for o in ref_outs]
    ref_idx = [sets_to_numpy(ref_sets[j]) for j in range(0, LAYERS, 2)]
    assert all(np.isfinite(r).all() for r in ref)

    runs = [fresh() for _ in range(ROUNDS)]
    for sets, outs in runs:  # every round enqueued before any host synchronisation
        _run(cases, ws, sets, outs, roles, sync_each=False)
    torch.cuda.synchronize()
    for sets, outs in runs:
        for j in range(LAYERS):
            np.testing.assert_array_equal(outs[j].cpu().numpy(), ref[j], err_msg=f"layer {j}")
        for k, j in enumerate(range(0, LAYERS, 2)):
            for a, b in zip(sets_to_numpy(sets[j]), ref_idx[k]):
                np.testing.assert_array_equal(a, b)
