"""Draft-tree utilities and the accepted-row commit (include/specsv_b200/
draft_tree.h) against the reference:

* the reference's own KATs (tests/test_draft_tree.cpp), restated through the
  C-ABI;
* golden vectors written by the compiled reference (tests/golden/
  draft_trees.npz, tests/golden/make_tree_golden.py) -- these run without
  /root/reference;
* live comparisons with the compiled reference (oracle/_ref) when present;
* the boundary's packed mask feeding the verify call, and (GPU) the commit of
  accepted rows followed by the compressed-block append, bit-exact.
"""
import os
import re

import numpy as np
import pytest

from paper_2605_19893_b200 import abi
from paper_2605_19893_b200 import tree as T
from paper_2605_19893_b200.abi import SpecsvError
from tests.tree_cases import CASES, arithmetic_proposer, argmax_for

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "specsv_b200", "draft_tree.h")
GOLDEN = os.path.join(HERE, "golden", "draft_trees.npz")
COMMITTED = 65536


def _prop(fn):
    return lambda node, tok, dep, cum, k: [T.TokenScore(t, s) for t, s in fn(node, tok, dep, cum, k)]


def example_tree():
    """r -> {a, b}, a -> {c, d}, b -> {e, f} (test_draft_tree.cpp:31-50)."""
    return T.DraftTree.from_nodes([(-1, 100, 0.0), (0, 1, -0.1), (0, 2, -0.2), (1, 3, -0.1),
                                   (1, 4, -0.2), (2, 5, -0.1), (2, 6, -0.2)])


def toks(tree, order):
    return [int(tree.token[i]) for i in order]


def test_library_exports_every_declared_symbol():
    decl = set(re.findall(r"\b(specsv_\w+)\s*\(", open(HEADER).read()))
    assert decl == set(T.EXPORTED)
    L = abi.lib()
    for name in T.EXPORTED:
        assert hasattr(L, name)


# ---- test_draft_tree.cpp ----------------------------------------------------
def test_expansion_node_counts():  # :57-78
    ar = _prop(arithmetic_proposer())
    t = T.expand_draft_tree(7, ar, 1, 1)
    assert t.gamma == 1 and t.depth[1] == 1
    assert T.expand_draft_tree(7, ar, 2, 2).gamma == 6
    assert T.expand_draft_tree(7, ar, 3, 3).gamma == (81 - 3) // 2
    t = T.expand_draft_tree(7, ar, 4, 3, 10)  # budget keeps ancestor closure
    assert t.gamma == 10
    for i in range(1, t.n_nodes):
        p = int(t.parent[i])
        assert 0 <= p < t.n_nodes and t.cum_score[p] >= t.cum_score[i]


def test_flatten_bfs_level_order_dfs_preorder():  # :80-99
    t = example_tree()
    bfs = T.flatten_tree(t, T.BFS, 50)
    dfs = T.flatten_tree(t, T.DFS, 50)
    assert toks(t, bfs.order) == [1, 2, 3, 4, 5, 6]
    assert toks(t, dfs.order) == [1, 3, 4, 2, 5, 6]
    assert bfs.positions.tolist() == [50, 50, 51, 51, 51, 51]
    assert dfs.positions.tolist() == [50, 51, 51, 50, 51, 51]
    chain = T.expand_draft_tree(7, _prop(arithmetic_proposer()), 4, 1)
    assert (T.flatten_tree(chain, T.BFS, 10).order == T.flatten_tree(chain, T.DFS, 10).order).all()


def test_tree_mask_kats():  # :101-146
    t = example_tree()
    dfs = T.flatten_tree(t, T.DFS, 50)
    m = dfs.mask_bool()
    assert m[1].tolist() == [True, True, False, False, False, False]
    assert m[2].tolist() == [True, False, True, False, False, False]
    chain = T.flatten_tree(T.expand_draft_tree(7, _prop(arithmetic_proposer()), 3, 1), T.BFS, 10)
    cm = chain.mask_bool()
    for i in range(3):
        for j in range(3):
            assert cm[i, j] == (j <= i)
    bfs = T.flatten_tree(t, T.BFS, 50)
    slot = {int(n): i for i, n in enumerate(dfs.order)}
    bm = bfs.mask_bool()
    for i, a in enumerate(bfs.order):
        for j, b in enumerate(bfs.order):
            assert bm[i, j] == m[slot[int(a)], slot[int(b)]]
    rng = np.random.default_rng(5)
    for trial in range(20):
        rt = T.expand_draft_tree(3, _prop(arithmetic_proposer(-0.01 * (trial + 1))), 3, 2,
                                 4 + int(rng.integers(8)))
        for trav in (T.BFS, T.DFS):
            fb = T.flatten_tree(rt, trav, 10)
            fm = fb.mask_bool()
            for i in range(fb.gamma):
                assert fm[i, i]
                for j in range(fb.gamma):
                    if fm[i, j]:
                        assert rt.is_ancestor_or_self(int(fb.order[j]), int(fb.order[i]))


def test_greedy_verify_kats():  # :148-178
    t = example_tree()
    vr = T.greedy_verify(t, [999] * 7)
    assert vr.accepted_tokens == [] and vr.bonus_token == 999 and vr.accepted_count == 1
    am = [999] * 7
    am[0], am[2], am[6] = 2, 6, 42
    vr = T.greedy_verify(t, am)
    assert vr.accepted_tokens == [2, 6] and vr.bonus_token == 42 and vr.accepted_count == 3
    assert vr.accepted_nodes == [2, 6]
    am = [999] * 7
    am[0], am[1] = 1, 77
    vr = T.greedy_verify(t, am)
    assert vr.accepted_tokens == [1] and vr.bonus_token == 77


# ---- error behaviour (std::invalid_argument in the reference) ------------------
def test_errors():
    ar = _prop(arithmetic_proposer())
    for D, k in ((0, 2), (2, 0)):
        with pytest.raises(SpecsvError) as e:
            T.expand_draft_tree(7, ar, D, k)
        assert e.value.code == abi.EINVAL
    with pytest.raises(SpecsvError):
        T.greedy_verify(example_tree(), [0] * 6)  # argmax missing for some nodes
    bad = example_tree()
    bad.depth = bad.depth.copy()
    bad.depth[3] = 5
    with pytest.raises(SpecsvError) as e:
        T.flatten_tree(bad, T.BFS, 10)
    assert e.value.code == abi.EINVAL
    with pytest.raises(SpecsvError):  # an ancestor missing from an explicit order
        T.build_tree_mask(example_tree(), [3, 4])
    with pytest.raises(SpecsvError):  # the proposer returns more than k
        T.expand_draft_tree(7, lambda n, t, d, c, k: [T.TokenScore(i, -i) for i in range(k + 1)], 2, 2)


# ---- golden vectors from the compiled reference ---------------------------------
def _golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_matches_reference_golden(ci):
    g = _golden()
    name, root, mk, D, k, budget = CASES[ci]
    pre = f"{name}/"
    t = T.expand_draft_tree(root, _prop(mk()), D, k, budget)
    assert t.parent.tolist() == g[pre + "parent"].tolist()
    assert t.token.tolist() == g[pre + "token"].tolist()
    assert t.depth.tolist() == g[pre + "depth"].tolist()
    assert np.array_equal(t.score, g[pre + "score"])
    assert np.array_equal(t.cum_score, g[pre + "cum"])
    for trav in (T.BFS, T.DFS):
        fb = T.flatten_tree(t, trav, COMMITTED)
        assert fb.order.tolist() == g[pre + f"order{trav}"].tolist()
        assert fb.positions.tolist() == g[pre + f"pos{trav}"].tolist()
        assert np.array_equal(fb.mask_bool(), g[pre + f"mask{trav}"].astype(bool))
        assert np.array_equal(T.build_tree_mask(t, fb.order), fb.mask)
    for s in range(3):
        vr = T.greedy_verify(t, g[pre + f"argmax{s}"])
        assert vr.accepted_nodes == g[pre + f"acc_nodes{s}"].tolist()
        assert vr.accepted_tokens == g[pre + f"acc_tokens{s}"].tolist()
        assert vr.bonus_token == int(g[pre + f"bonus{s}"][0])


def test_live_against_compiled_reference():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    ref = O.RefTree()
    from tests.tree_cases import hashed_proposer
    for seed in range(12):
        D, k = 2 + seed % 5, 1 + seed % 4
        budget = None if seed % 3 == 0 else 5 + 3 * seed
        rc, (parent, token, depth, score, cum) = ref.expand(seed + 2, hashed_proposer(50 + seed), D, k,
                                                            budget)
        assert rc == 0
        t = T.expand_draft_tree(seed + 2, _prop(hashed_proposer(50 + seed)), D, k, budget)
        assert t.parent.tolist() == parent.tolist() and t.token.tolist() == token.tolist()
        for trav in (T.BFS, T.DFS):
            order, pos, mask = ref.flatten(parent, token, depth, score, trav, 1000 + seed)
            fb = T.flatten_tree(t, trav, 1000 + seed)
            assert fb.order.tolist() == order.tolist() and fb.positions.tolist() == pos.tolist()
            assert np.array_equal(fb.mask_bool(), mask)
        am = argmax_for(parent, token, seed)
        _, nodes, tks, bonus = ref.greedy(parent, token, depth, score, am)
        vr = T.greedy_verify(t, am)
        assert (vr.accepted_nodes, vr.accepted_tokens, vr.bonus_token) == (nodes, tks, bonus)


def test_flattened_mask_is_the_boundary_format():
    """flatten_tree's packed mask equals workload.tree_mask_from_parents for the
    same flat order (the layout the verify call and the oracle read)."""
    from paper_2605_19893_b200.workload import tree_mask_from_parents
    g = _golden()
    name = "c3_d6k4_b32/"
    t = T.DraftTree(g[name + "parent"], g[name + "token"], g[name + "depth"], g[name + "score"])
    for trav in (T.BFS, T.DFS):
        fb = T.flatten_tree(t, trav, COMMITTED)
        slot = {int(n): i for i, n in enumerate(fb.order)}
        parents = [-1 if int(t.parent[n]) == 0 else slot[int(t.parent[n])] for n in fb.order]
        assert np.array_equal(fb.mask, tree_mask_from_parents(parents))


# ---- commit of accepted rows (GPU) -------------------------------------------
@pytest.mark.gpu
def test_commit_accepted_rows_then_compress(oracle_lib):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O
    from paper_2605_19893_b200 import verify as V
    from paper_2605_19893_b200.workload import LayerInputs, bf16_round
    cfg = O.llama_config(3)
    vcfg = V.NsaConfig(**cfg.__dict__)
    rows0, gamma, cap = 1020, 12, 1100  # the commit completes block 62
    xs = [LayerInputs(cfg, rows0, gamma, 40 + j) for j in range(3)]
    pes = [torch.from_numpy(x.pos_embed).cuda() for x in xs]
    caches, tks, tvs = [], [], []
    for x, pe in zip(xs, pes):
        c = V.LayerCache(vcfg, cap)
        c.append(torch.from_numpy(x.k).cuda().bfloat16(), torch.from_numpy(x.v).cuda().bfloat16())
        c.extend_compressed(pe)
        caches.append(c)
        tks.append(torch.from_numpy(x.tree_k[:gamma]).cuda().bfloat16())
        tvs.append(torch.from_numpy(x.tree_v[:gamma]).cuda().bfloat16())
    slots = [3, 7, 8, 11]  # an accepted root-to-leaf path in flat slots
    T.commit_accepted(vcfg, caches, tks, tvs, slots, pos_embed=pes)
    torch.cuda.synchronize()
    for j, (x, c) in enumerate(zip(xs, caches)):
        assert c.rows == rows0 + len(slots)
        want_k = np.concatenate([bf16_round(x.k), bf16_round(x.tree_k[slots])])
        want_v = np.concatenate([bf16_round(x.v), bf16_round(x.tree_v[slots])])
        assert np.array_equal(c.k[:c.rows].float().cpu().numpy(), want_k)
        assert np.array_equal(c.v[:c.rows].float().cpu().numpy(), want_v)
        assert np.array_equal(c.k[c.rows:].float().cpu().numpy(), np.zeros_like(c.k[c.rows:].cpu().float().numpy()))
        ck, _ = oracle_lib.build_compressed(cfg, want_k, want_v, c.rows, x.pos_embed)
        assert c.blocks == ck.shape[0] == vcfg.compressed_block_count(rows0) + 1
        assert np.array_equal(c.ck[:c.blocks].cpu().numpy().view(np.uint32), ck.view(np.uint32))
    with pytest.raises(SpecsvError):  # beyond the cache capacity
        T.commit_accepted(vcfg, caches, tks, tvs, list(range(12)) * 9, pos_embed=pes)
