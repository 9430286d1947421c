"""GPU parity of the verify path on C3 as specified: the draft
tree comes from expand_draft_tree (D=6, k=4, budget 32, the hashed proposer
of tests/tree_cases.py) flattened in BFS and DFS order at 64K context; and
the near-tie contract P2 of tests/test_gpu_parity.py exercised on a
constructed exact tie at the Top-n boundary.  All calls through the C-ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import tree as T  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs, tree_mask_from_parents  # noqa: E402
from tests import tree_cases  # noqa: E402
from tests.gpu_harness import TOL, DeviceCase, rel_errors, sets_to_numpy  # noqa: E402
from tests.test_gpu_parity import NEAR_TIE, _check_indices  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def c3_flat(traversal, committed):
    name, root, prop, D, k, budget = [c for c in tree_cases.CASES if c[0] == "c3_d6k4_b32"][0]
    pf = prop()
    tree = T.expand_draft_tree(root, lambda *a: [T.TokenScore(t, sc) for t, sc in pf(*a)], D, k, budget)
    flat = T.flatten_tree(tree, traversal, committed)
    slot = {int(node): i for i, node in enumerate(flat.order)}
    parents = [slot.get(int(tree.parent[int(node)]), -1) for node in flat.order]
    return tree, flat, parents


@pytest.mark.parametrize("traversal", [T.BFS, T.DFS])
def test_c3_expanded_tree_64k(oracle_lib, traversal):
    """C3: the expanded 32-node tree at 64K, refresh (exact and approx) then a
    reuse layer inheriting the exact sets, against the oracle; the flattened
    positions and packed mask are the ones specsv_tree_flatten produces."""
    cfg = O.llama_config(32)
    ctx = 65536
    tree, flat, parents = c3_flat(traversal, ctx)
    assert flat.gamma == 32 and int(tree.depth.max()) <= cfg.routing_lag
    x = LayerInputs(cfg, ctx, flat.gamma, 6400 + traversal, parent_slot=parents)
    assert np.array_equal(x.pos[1:], flat.positions)
    assert np.array_equal(x.tree_mask, flat.mask)
    assert np.array_equal(tree_mask_from_parents(parents), flat.mask)
    case = DeviceCase(cfg, x)
    for mode in (O.MODE_EXACT, O.MODE_APPROX):
        out, sets = case.run(4, mode, V.ROLE_REFRESH)
        ref = case.oracle(oracle_lib, 4, mode, O.ROLE_REFRESH)
        assert ref["rc"] == 0
        gi, gc, gf = sets_to_numpy(sets)
        assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
        per, l2 = rel_errors(out, ref["out"])
        assert per <= TOL and l2 <= TOL, (mode, per, l2)
        if mode == O.MODE_EXACT:
            exact_sets, exact_ref = sets, ref
    y = LayerInputs(cfg, ctx, flat.gamma, 6500 + traversal, parent_slot=parents)
    case2 = DeviceCase(cfg, y)
    out2, _ = case2.run(4, V.MODE_EXACT, V.ROLE_REUSE, sets=exact_sets)
    ref2 = case2.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REUSE, idx=exact_ref["idx"],
                        idx_count=exact_ref["idx_count"], idx_forced=exact_ref["idx_forced"])
    per, l2 = rel_errors(out2, ref2["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_near_tie_at_the_topn_boundary(oracle_lib):
    """An exact tie at the Top-n boundary, constructed by copying the key rows
    around the last selected non-forced block b1 onto another block b2 (same
    offset inside its 16-block routing tile, so both see the same compressed
    keys): the oracle's scores of b1 and b2 are bit-identical and the lower id
    wins.  The GPU's fp64 scores may differ from each other by rounding (P3),
    so either block may come out; P2 accepts exactly such a flip (boundary gap
    <= NEAR_TIE) and nothing else -- checked on the device result and on a
    simulated flip at the tie and at a non-tie position."""
    cfg = O.llama_config(4)
    rows = 8192
    x = LayerInputs(cfg, rows, 4, 777)
    ck, _ = oracle_lib.build_compressed(cfg, x.k, x.v, rows, x.pos_embed)
    vis = cfg.routing_visible_len(int(x.pos[0]))
    s = oracle_lib.selection_scores(cfg, x.q[0], ck, vis)
    avail = s.size
    forced = {0, avail - 2, avail - 1}
    order = [b for b in np.argsort(-s, kind="stable") if b not in forced]
    want = cfg.n - len(forced)
    b1 = int(order[want - 1])  # the last selected non-forced block
    k0 = x.k.copy()
    lo = 64 * b1 - cfg.d
    # an unselected block at the same tile offset, away from b1 and the forced
    # ones, whose copy lands the tie on the boundary (the copy also moves the
    # softmax normalisation, so try candidates until it does)
    for b2 in (int(b) for b in order[want + 40:]):
        if b2 % 4 != b1 % 4 or abs(b2 - b1) <= 4 or not 2 < b2 < avail - 4:
            continue
        x.k = k0.copy()
        x.k[64 * b2 - cfg.d:64 * b2 + 64 + cfg.d] = k0[lo:lo + 64 + 2 * cfg.d]
        ck, _ = oracle_lib.build_compressed(cfg, x.k, x.v, rows, x.pos_embed)
        s = oracle_lib.selection_scores(cfg, x.q[0], ck, vis)
        assert s[b1] == s[b2]
        sel = oracle_lib.select_blocks(cfg, s, cfg.n, vis)[0]
        if (b1 in sel) != (b2 in sel):
            break
    else:
        pytest.fail("no boundary tie constructed")
    case = DeviceCase(cfg, x)
    ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
    r0 = list(ref["idx"][0, :ref["idx_count"][0]])
    assert (b1 in r0) != (b2 in r0) and min(b1, b2) in r0  # a boundary tie, lower id wins
    out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    near = _check_indices(oracle_lib, case, gi, gc, gf, ref)
    assert near <= case.nq
    per, l2 = rel_errors(out, ref["out"])
    assert per <= 2 * TOL and l2 <= TOL, (per, l2)  # a flipped block moves one query's slc branch
    # the exemption accepts the tie flip ...
    fi = ref["idx"].astype(np.int64).copy()
    fc = ref["idx_count"].astype(np.int64).copy()
    ff = np.array([sum(1 << i for i in range(cfg.n) if ref["idx_forced"][q, i]) for q in range(case.nq)],
                  np.int64)
    row = sorted((set(r0) - {min(b1, b2)}) | {max(b1, b2)})
    fi[0, :len(row)] = row
    ff[0] = sum(1 << i for i, b in enumerate(row) if b in forced)
    assert _check_indices(oracle_lib, case, fi, fc, ff, ref) == 1
    # ... and nothing else
    other = [b for b in range(3, avail - 3) if b not in r0 and b not in (b1, b2)][0]
    bad = sorted((set(r0) - {int(order[0])}) | {other})
    fi2 = ref["idx"].astype(np.int64).copy()
    fi2[0, :len(bad)] = bad
    with pytest.raises(AssertionError):
        _check_indices(oracle_lib, case, fi2, fc, ff, ref)
    assert NEAR_TIE == 1e-12
