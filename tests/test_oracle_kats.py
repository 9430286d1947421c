"""Known-answer tests of the reference, replayed against BOTH the C oracle and
the compiled reference (``impl`` fixture).  Each test cites the reference
test it restates (paths relative to /root/reference/proj/tests)."""
import math

import numpy as np
import pytest

from oracle.oracle import NsaConfig, small_config
from paper_2605_19893_b200.workload import splitmix_symmetric, splitmix_unit


def rand_kv(seed, cfg, rows):
    k = splitmix_symmetric(seed, 1.0, rows * cfg.n_kv_heads * cfg.d_head)
    v = splitmix_symmetric(seed + 1, 1.0, rows * cfg.n_kv_heads * cfg.d_head)
    return (k.reshape(rows, cfg.n_kv_heads, cfg.d_head), v.reshape(rows, cfg.n_kv_heads, cfg.d_head))


def rand_q(seed, cfg):
    return splitmix_symmetric(seed, 1.0, cfg.n_q_heads * cfg.d_head).reshape(cfg.n_q_heads, cfg.d_head)


def normalized(p):
    dh = p.shape[-1] - 2
    den = p[..., dh + 1:dh + 2]
    return np.where(den == 0, 0.0, p[..., :dh] / np.where(den == 0, 1, den))


def dense_oracle(qh, keys, vals):
    """test_util.hpp:56-80 two-pass softmax."""
    if len(keys) == 0:
        return np.zeros(len(qh))
    scale = 1.0 / math.sqrt(len(qh))
    logits = np.array([np.dot(qh.astype(np.float64), k.astype(np.float64)) * scale for k in keys])
    w = np.exp(logits - logits.max())
    w /= w.sum()
    return (w[:, None] * np.array(vals, np.float64)).sum(0)


def test_config_invariants(impl):  # test_nsa_core.cpp:15-31
    cfg = NsaConfig()
    assert impl.validate(cfg)
    for field, val in (("d", cfg.l + 1), ("l_sel", cfg.d + 1), ("n", 2), ("n_q_heads", 3)):
        bad = NsaConfig(**{**cfg.__dict__, field: val})
        assert not impl.validate(bad)
    assert not impl.validate(NsaConfig(w=8, routing_lag=16))


def test_compressed_block_count(impl):  # test_nsa_core.cpp:33-39
    cfg = NsaConfig(l=32, d=16)
    assert impl.compressed_block_count(64, cfg) == 3
    assert impl.compressed_block_count(31, cfg) == 0
    assert impl.compressed_block_count(32, cfg) == 1


def test_pooling_ranges(impl):  # test_nsa_core.cpp:41-65
    cfg = small_config()
    k, v = rand_kv(21, cfg, 16)
    pe = splitmix_symmetric(99, 0.2, cfg.l * cfg.d_head).reshape(cfg.l, cfg.d_head)
    ck, cv = impl.build_compressed(cfg, k, v, 16, pe)
    assert ck.shape[0] == 3
    for b in range(3):
        rows = slice(b * cfg.d, b * cfg.d + cfg.l)
        mk = (k[rows, 0].astype(np.float64) + pe.astype(np.float64)).mean(0)
        mv = v[rows, 0].astype(np.float64).mean(0)
        np.testing.assert_allclose(ck[b, 0], mk, rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(cv[b, 0], mv, rtol=1e-5, atol=1e-7)


def test_scores_singleton_and_symmetry(impl):  # test_nsa_core.cpp:67-102
    cfg = small_config()
    k, v = rand_kv(22, cfg, cfg.l)
    ck, cv = impl.build_compressed(cfg, k, v, cfg.l)
    s = impl.selection_scores(cfg, rand_q(5, cfg), ck, cfg.l)
    assert abs(s.sum() - 1.0) <= 1e-12
    c2 = NsaConfig(**{**cfg.__dict__, "l_sel": cfg.l})
    krow = splitmix_symmetric(7, 1.0, c2.d_head)
    rows = c2.l + c2.d
    k = np.tile(krow, (rows, 1)).reshape(rows, 1, c2.d_head)
    v = splitmix_symmetric(8, 1.0, rows * c2.d_head).reshape(rows, 1, c2.d_head)
    ck, cv = impl.build_compressed(c2, k, v, rows)
    assert ck.shape[0] == 2
    s = impl.selection_scores(c2, rand_q(9, c2), ck, rows)
    assert s.shape == (2,)
    assert abs(s[0] - 0.75) <= 1e-12 and abs(s[1] - 0.25) <= 1e-12


def test_scores_dense_oracle(impl):  # test_nsa_core.cpp:104-150
    cfg = small_config()
    N = 256
    k, v = rand_kv(23, cfg, N)
    pe = splitmix_symmetric(24, 0.2, cfg.l * cfg.d_head).reshape(cfg.l, cfg.d_head)
    ck, cv = impl.build_compressed(cfg, k, v, N, pe)
    q = rand_q(25, cfg)
    s = impl.selection_scores(cfg, q, ck, N)
    m = min((N - cfg.l) // cfg.d + 1, ck.shape[0])
    scale = 1 / math.sqrt(cfg.d_head)
    mass = np.zeros(m)
    for h in range(cfg.n_q_heads):
        lg = ck[:m, h // (cfg.n_q_heads // cfg.n_kv_heads)].astype(np.float64) @ q[h].astype(np.float64) * scale
        e = np.exp(lg - lg.max())
        mass += e / e.sum()
    expect = np.zeros(-(-N // cfg.l_sel))
    for i in range(m):
        lo, hi = i * cfg.d, i * cfg.d + cfg.l
        b = lo // cfg.l_sel
        while b * cfg.l_sel < hi:
            olo, ohi = max(lo, b * cfg.l_sel), min(hi, (b + 1) * cfg.l_sel)
            if ohi > olo:
                expect[b] += mass[i] / cfg.n_q_heads * (ohi - olo) / cfg.l
            b += 1
    np.testing.assert_allclose(s, expect, rtol=1e-10)


def test_select_blocks_kat(impl):  # test_nsa_core.cpp:152-161
    cfg = NsaConfig(l_sel=64, d=16)
    idx, forced = impl.select_blocks(cfg, [0.9, 0.1, 0.8, 0.2, 0.7], 3, 5 * 64, forced=[0, 4])
    assert idx == [0, 2, 4]
    assert forced == [True, False, True]


def test_select_blocks_supply_below_n(impl):  # test_nsa_core.cpp:163-168
    cfg = small_config()
    idx, _ = impl.select_blocks(cfg, [0.3, 0.7], 16, 2 * cfg.l_sel)
    assert idx == [0, 1]


def test_select_blocks_forced_floor(impl):  # test_nsa_core.cpp:170-187
    cfg = small_config()
    vis = 8 * cfg.l_sel
    for t in range(50):
        a, _ = impl.select_blocks(cfg, splitmix_unit(1000 + t, 8), cfg.n, vis)
        b, _ = impl.select_blocks(cfg, splitmix_unit(2000 + t, 8), cfg.n, vis)
        assert len(set(a) & set(b)) >= 3


def test_select_blocks_ties_go_to_lower_id(impl):  # nsa_attention.cpp:120-123
    cfg = NsaConfig(l_sel=64, d=16)
    idx, _ = impl.select_blocks(cfg, [0.5] * 10, 5, 10 * 64)
    assert idx == [0, 1, 2, 8, 9]


def test_compressed_branch_cases(impl):  # test_nsa_core.cpp:189-231
    cfg = small_config()
    k, v = rand_kv(25, cfg, cfg.l)
    ck, cv = impl.build_compressed(cfg, k, v, cfg.l)
    q = rand_q(26, cfg)
    p = impl.branch_compressed(cfg, q, ck, cv, cfg.l - 1)
    assert (p[:, -1] == 0).all() and (p[:, :-2] == 0).all()
    p = impl.branch_compressed(cfg, q, ck, cv, cfg.l)
    assert (normalized(p) == cv[0, 0].astype(np.float64)).all()
    k, v = rand_kv(27, cfg, cfg.l + 2 * cfg.d)
    ck, cv = impl.build_compressed(cfg, k, v, cfg.l + 2 * cfg.d)
    p = impl.branch_compressed(cfg, q, ck, cv, cfg.l + 2 * cfg.d)
    for h in range(cfg.n_q_heads):
        o = dense_oracle(q[h], list(ck[:3, 0]), list(cv[:3, 0]))
        assert np.abs(normalized(p)[h] - o).max() <= 1e-12


def test_selected_branch_ownership_exact(impl):  # test_nsa_core.cpp:233-286
    cfg = small_config()
    N = 4 * cfg.l_sel
    k, v = rand_kv(26, cfg, N)
    q = rand_q(27, cfg)
    p = impl.branch_selected(cfg, q, k, v, [], N)
    assert (p[:, -1] == 0).all()
    p = impl.branch_selected(cfg, q, k, v, [0, 1, 2, 3], N)
    for h in range(cfg.n_q_heads):
        o = dense_oracle(q[h], list(k[:, 0]), list(v[:, 0]))
        assert np.abs(normalized(p)[h] - o).max() <= 1e-12
    masked = impl.branch_selected(cfg, q, k, v, [0, 1, 2, 3], N, ownership=[1, 0, 1, 1])
    plain = impl.branch_selected(cfg, q, k, v, [0, 2, 3], N)
    assert (masked == plain).all()  # bit-identical
    bounded = impl.branch_selected(cfg, q, k, v, [0, 3], cfg.l_sel)
    first = impl.branch_selected(cfg, q, k, v, [0], cfg.l_sel)
    assert (normalized(bounded) == normalized(first)).all()


def test_window_ranges_and_tree_rows(impl):  # test_nsa_core.cpp:288-342
    cfg = NsaConfig(**{**small_config().__dict__, "w": 512})
    k, v = rand_kv(27, cfg, 128)
    q = rand_q(28, cfg)
    p = impl.branch_window(cfg, q, k, v, 100, 128)
    for h in range(cfg.n_q_heads):
        o = dense_oracle(q[h], list(k[:101, 0]), list(v[:101, 0]))
        assert np.abs(normalized(p)[h] - o).max() <= 1e-12
    k, v = rand_kv(29, cfg, 1001)
    p = impl.branch_window(cfg, q, k, v, 1000, 1001)
    for h in range(cfg.n_q_heads):
        o = dense_oracle(q[h], list(k[489:1001, 0]), list(v[489:1001, 0]))
        assert np.abs(normalized(p)[h] - o).max() <= 1e-12
    c = 64
    k, v = rand_kv(30, cfg, c)
    tk, tv = rand_kv(31, cfg, 3)
    p = impl.branch_window(cfg, q, k, v, c + 1, c, tk, tv, [0, 2])
    for h in range(cfg.n_q_heads):
        keys = list(k[:, 0]) + [tk[0, 0], tk[2, 0]]
        vals = list(v[:, 0]) + [tv[0, 0], tv[2, 0]]
        assert np.abs(normalized(p)[h] - dense_oracle(q[h], keys, vals)).max() <= 1e-12


def test_merge_partials(impl):  # test_nsa_core.cpp:344-386
    cfg = small_config()
    N = 40
    k, v = rand_kv(28, cfg, N)
    q = rand_q(29, cfg)
    whole = list(range(-(-N // cfg.l_sel)))
    full = impl.branch_selected(cfg, q, k, v, whole, N)
    empty = np.zeros(cfg.d_head + 2)
    empty[-2] = -np.inf
    m = impl.merge_partials(full[0], empty)
    assert m[-1] == full[0, -1] and (m[:-2] == full[0, :-2]).all()
    for split in range(1, len(whole)):
        pl = impl.branch_selected(cfg, q, k, v, whole[:split], N)
        ph = impl.branch_selected(cfg, q, k, v, whole[split:], N)
        for h in range(cfg.n_q_heads):
            mg = impl.merge_partials(pl[h], ph[h])
            assert np.abs(normalized(mg) - normalized(full[h])).max() <= 1e-12
    pl = impl.branch_selected(cfg, q, k, v, [0], N)
    ph = impl.branch_selected(cfg, q, k, v, [1, 2], N)
    for h in range(cfg.n_q_heads):
        ab, ba = impl.merge_partials(pl[h], ph[h]), impl.merge_partials(ph[h], pl[h])
        assert ab[-1] == ba[-1] and (ab[:-2] == ba[:-2]).all()


def test_gated_combine(impl):  # test_nsa_core.cpp:388-421
    cfg = small_config()
    k, v = rand_kv(29, cfg, 32)
    q = rand_q(30, cfg)
    cmp = impl.branch_selected(cfg, q, k, v, [0], 32)[0]
    slc = impl.branch_selected(cfg, q, k, v, [1], 32)[0]
    win = impl.branch_window(cfg, q, k, v, 31, 32)[0]
    out = impl.gated_combine(cmp, slc, win, [0.0, 0.0, 1.0])
    assert (out == normalized(win)).all()
    e = np.zeros(cfg.d_head + 2)
    e[-2] = -np.inf
    assert (impl.gated_combine(e, e, e, [0.9, 0.9, 0.9]) == 0).all()
    g = [0.3, 0.5, 0.7]
    out = impl.gated_combine(cmp, slc, win, g)
    expect = g[0] * normalized(cmp) + g[1] * normalized(slc) + g[2] * normalized(win)
    np.testing.assert_allclose(out, expect, rtol=1e-14)


def test_merged_schedule_kat(impl):  # test_grouped_verifier.cpp:106-131
    u, own = impl.merged_schedule([[0, 2, 5, 7], [0, 3, 5, 8]])
    assert u == [0, 2, 3, 5, 7, 8]
    assert own[0] == [True, True, False, True, True, False]
    assert own[1] == [True, False, True, True, False, True]
    u, _ = impl.merged_schedule([[0, 2, 5, 7], [0, 2, 5, 7]])
    assert u == [0, 2, 5, 7]
    u, _ = impl.merged_schedule([[0, 1, 2, 14, 15], [0, 5, 6, 14, 15], [0, 9, 10, 14, 15]])
    assert 15 - len(u) == 3 * 2


def test_representative_index(impl):  # test_grouped_verifier.cpp:205-214
    assert impl.representative_index([100, 100, 100]) == 2
    assert impl.representative_index([100, 103, 101]) == 1


def test_clamp_kats(impl):  # test_fusion_schedule.cpp:56-80
    cfg = NsaConfig(l_sel=64)
    src, fl = [0, 2, 5, 9], [1, 0, 0, 1]
    assert impl.clamp_inherited(cfg, src, fl, 10 * 64) == (src, [True, False, False, True])
    assert impl.clamp_inherited(cfg, src, fl, 5 * 64 + 10)[0] == [0, 2, 5]
    assert impl.clamp_inherited(cfg, src, fl, 64) == ([0], [True])


def test_dot_matches_long_double(impl):  # test_kernels.cpp:27-38
    for n in (0, 1, 3, 4, 7, 64, 129):
        a = splitmix_symmetric(11 + n, 3.0, n)
        b = splitmix_symmetric(12 + n, 3.0, n)
        ref = float(np.sum(np.longdouble(a) * np.longdouble(b)))
        assert abs(impl.dot(a, b) - ref) <= 1e-10 * (1 + abs(ref))
