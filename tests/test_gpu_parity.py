"""GPU parity of the sm_100a verify path against the CPU oracle (the C
restatement pinned bit-exact to the reference).  All calls go through the
C-ABI.  Contract:
  P1  Top-n fed the oracle's fp64 scores returns identical indices/flags.
  P2  end-to-end indices equal the oracle's for every query whose oracle
      boundary gap exceeds NEAR_TIE (near-ties are counted, expected 0).
  P3  fp64 scores within 1e-13 relative of the oracle.
  P4  outputs within 2e-3: per (query, head) inf-norm relative and global L2.
  P5  LoadStats integers equal (test_abi_cpu covers the host accounting).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs, bf16_round  # noqa: E402
from tests.gpu_harness import (TOL, DeviceCase, boundary_gap, diff_within_near_tie,  # noqa: E402
                               forced_matrix, rel_errors, sets_to_numpy)

NEAR_TIE = 1e-12
TREE8 = [-1, -1, 0, 0, 1, 2, 2, 4]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check_indices(oracle_lib, case, got_idx, got_cnt, got_forced, ref, routed_only=None):
    cfg = case.cfg
    ck, _ = case.oracle_cache(oracle_lib)
    near = 0
    for q in range(case.nq):
        if ref["idx_count"][q] < 0:
            assert got_cnt[q] == -1, f"query {q} should have no set"
            continue
        nf = min(got_cnt[q], 32)  # the ABI's forced mask holds positions 0..31 (nsa_verify.h)
        same = (got_cnt[q] == ref["idx_count"][q]
                and (got_idx[q, :got_cnt[q]] == ref["idx"][q, :got_cnt[q]]).all()
                and (forced_matrix(got_forced[q:q + 1], cfg.n)[0, :nf]
                     == ref["idx_forced"][q, :nf]).all())
        if not same:
            gap = boundary_gap(oracle_lib, cfg, case.x.q[q], ck, case.x.pos[q])
            assert gap <= NEAR_TIE, f"query {q}: indices differ with gap {gap}"
            # and only by blocks at that near-tie
            assert diff_within_near_tie(oracle_lib, cfg, case.x.q[q], ck, case.x.pos[q],
                                        got_idx[q, :max(got_cnt[q], 0)],
                                        ref["idx"][q, :ref["idx_count"][q]], NEAR_TIE), \
                f"query {q}: indices differ beyond the near-tie"
            near += 1
    return near


def test_compress_append_bit_exact(oracle_lib):
    cfg = O.llama_config(2)
    x = LayerInputs(cfg, 3000, 0, 5)
    case = DeviceCase(cfg, x)
    ck, cv = oracle_lib.build_compressed(cfg, x.k, x.v, 3000, x.pos_embed)
    nb = ck.shape[0]
    assert case.cache.blocks == nb
    got_ck = case.cache.ck[:nb].cpu().numpy()
    assert np.array_equal(got_ck.view(np.uint32), ck.view(np.uint32))
    got_cv = case.cache.cv[:nb].float().cpu().numpy()
    assert np.array_equal(got_cv, bf16_round(cv))
    got_ck16 = case.cache.ck16[:nb].float().cpu().numpy()
    assert np.array_equal(got_ck16, bf16_round(ck))


def test_compress_digit_planes():
    """The routing keys' digit planes (ABI v3) written by the compressed append:
    per (block, head) row, e is the smallest power of two above max |ck|, the
    four signed base-256 digits recombine to round(ck 2^(30 - e)), and ckexp
    also counts the elements that rounding changed."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 3000, 2, 77)
    case = DeviceCase(cfg, x)
    c = case.cache
    nb = c.blocks
    ck = c.ck[:nb].cpu().numpy().astype(np.float64)
    packed = c.ckexp[:nb].cpu().numpy().astype(np.int64)
    e = ((packed & 0xFFFF) ^ 0x8000) - 0x8000  # low 16 bits, signed
    nrounded = (packed >> 16) & 0xFF
    dg = c.ckd[:nb].cpu().numpy().astype(np.int64)  # [nb][H][4][dh]
    X = dg[:, :, 0] + 256 * dg[:, :, 1] + 65536 * dg[:, :, 2] + 16777216 * dg[:, :, 3]
    mx = np.abs(ck).max(-1)
    assert (mx < np.ldexp(1.0, e)).all() and (mx >= np.ldexp(1.0, e - 1)).all()
    scaled = ck * np.ldexp(1.0, 30 - e)[..., None]
    want = np.rint(scaled)
    assert np.array_equal(X, want.astype(np.int64))
    assert np.array_equal(nrounded, (want != scaled).sum(-1))  # the elements the grid rounds
    assert dg.min() >= -128 and dg.max() <= 127


def test_compress_append_incremental(oracle_lib):
    cfg = O.llama_config(2)
    x = LayerInputs(cfg, 2000, 0, 6)
    vcfg = V.NsaConfig(**cfg.__dict__)
    cache = V.LayerCache(vcfg, 2000)
    pe = torch.from_numpy(x.pos_embed).cuda()
    for lo, hi in ((0, 40), (40, 47), (47, 1000), (1000, 2000)):
        cache.append(torch.from_numpy(x.k[lo:hi]).cuda().bfloat16(),
                     torch.from_numpy(x.v[lo:hi]).cuda().bfloat16())
        cache.extend_compressed(pe)
    ck, _ = oracle_lib.build_compressed(cfg, x.k, x.v, 2000, x.pos_embed)
    assert np.array_equal(cache.ck[:ck.shape[0]].cpu().numpy().view(np.uint32), ck.view(np.uint32))


@pytest.mark.parametrize("rows", [700, 4096, 9000])
def test_selection_scores_fp64(oracle_lib, rows):
    cfg = O.llama_config(2)
    x = LayerInputs(cfg, rows, 3, 7 + rows)
    case = DeviceCase(cfg, x)
    ck, _ = case.oracle_cache(oracle_lib)
    for q in range(case.nq):
        got = V.selection_scores(case.vcfg, case.cache, case.batch, q, case.ws).cpu().numpy()
        ref = oracle_lib.selection_scores(cfg, x.q[q], ck, cfg.routing_visible_len(int(x.pos[q])))
        assert got.shape == ref.shape
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_select_blocks_on_reference_scores(oracle_lib):
    cfg = O.llama_config(2)
    vcfg = V.NsaConfig(**cfg.__dict__)
    rng = np.random.default_rng(3)
    for avail in (1, 2, 3, 5, 16, 17, 100, 1024, 2048):
        for trial in range(3):
            s = rng.random(avail)
            if trial == 2:
                s = np.round(s * 8) / 8  # many exact ties -> lower id wins
            vis = avail * cfg.l_sel
            ref = oracle_lib.select_blocks(cfg, s, cfg.n, vis)
            got = V.select_blocks(vcfg, torch.from_numpy(s).cuda(), vis)
            assert got == ref, (avail, trial)


CASES = [
    # rows, gamma, parents, mode, C
    (1000, 0, None, O.MODE_EXACT, 1),
    (1000, 4, None, O.MODE_EXACT, 2),
    (4096, 4, None, O.MODE_EXACT, 4),   # C1 shape
    (2085, 8, None, O.MODE_APPROX, 4),
    (3001, 8, TREE8, O.MODE_EXACT, 2),
    (3001, 8, TREE8, O.MODE_APPROX, 4),
    (9000, 8, None, O.MODE_EXACT, 8),
    (520, 3, None, O.MODE_EXACT, 1),    # window covers the whole context
    (40, 2, None, O.MODE_EXACT, 1),     # almost nothing compressed / selectable
]


@pytest.mark.parametrize("rows,gamma,parents,mode,C", CASES)
def test_verify_refresh_then_reuse(oracle_lib, rows, gamma, parents, mode, C):
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, rows, gamma, 100 + rows + gamma, parent_slot=parents)
    case = DeviceCase(cfg, x)
    out, sets = case.run(C, mode, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, C, mode, O.ROLE_REFRESH)
    assert ref["rc"] == 0
    gi, gc, gf = sets_to_numpy(sets)
    near = _check_indices(oracle_lib, case, gi, gc, gf, ref)
    assert near == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)

    # reuse layer: different KV, inherits the refresh layer's sets
    y = LayerInputs(cfg, rows, gamma, 900 + rows + gamma, parent_slot=parents)
    case2 = DeviceCase(cfg, y)
    out2, _ = case2.run(C, mode, V.ROLE_REUSE, sets=sets)
    ref2 = case2.oracle(oracle_lib, C, mode, O.ROLE_REUSE, idx=ref["idx"],
                        idx_count=ref["idx_count"], idx_forced=ref["idx_forced"])
    assert ref2["rc"] == 0
    per, l2 = rel_errors(out2, ref2["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_64k_chain8_full_size(oracle_lib):
    """Config C2 at full size (65536 committed rows, 8-token chain), one layer."""
    cfg = O.llama_config(32)
    x = LayerInputs(cfg, 65536, 8, 4242)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_tree32(oracle_lib):
    """Config C3 shape: 32-node tree (D <= 6) at 8K context, BFS flat order."""
    cfg = O.llama_config(4)
    parents = [-1, -1, -1, -1]
    for i in range(4, 32):
        parents.append(i // 4 - 1 if i // 4 - 1 < i else -1)
    # depths stay <= 6 <= routing_lag
    x = LayerInputs(cfg, 8192, 32, 77, parent_slot=parents)
    case = DeviceCase(cfg, x)
    for mode, C in ((O.MODE_EXACT, 4), (O.MODE_APPROX, 4)):
        out, sets = case.run(C, mode, V.ROLE_REFRESH)
        ref = case.oracle(oracle_lib, C, mode, O.ROLE_REFRESH)
        gi, gc, gf = sets_to_numpy(sets)
        assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
        per, l2 = rel_errors(out, ref["out"])
        assert per <= TOL and l2 <= TOL, (mode, per, l2)


def test_deterministic(oracle_lib):
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 5000, 8, 31)
    case = DeviceCase(cfg, x)
    a, _ = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    b, _ = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    assert np.array_equal(a, b)


def test_depth_beyond_lag_rejected():
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 2000, 2, 3)
    case = DeviceCase(cfg, x)
    case.batch.pos = case.batch.pos.copy()
    case.batch.pos[2] = case.batch.pos[0] + cfg.routing_lag + 1
    with pytest.raises(V.SpecsvError) as e:
        case.run(1, V.MODE_EXACT, V.ROLE_REFRESH)
    assert e.value.code == 1


def test_robust_redo_pass_forced(oracle_lib, monkeypatch):
    """The attend kernel's robust (running-max) pass, forced for every CTA,
    matches the oracle like the fast fixed-reference pass does."""
    monkeypatch.setenv("SPECSV_ATTEND_FORCE_ROBUST", "1")
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 3001, 8, 3109, parent_slot=TREE8)
    case = DeviceCase(cfg, x)
    out, sets = case.run(2, V.MODE_EXACT, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 2, O.MODE_EXACT, O.ROLE_REFRESH)
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


@pytest.mark.parametrize("scale", [30.0, 0.001])
def test_extreme_logit_ranges(oracle_lib, scale):
    """Queries scaled so logits span far more than the fast pass's +-48
    (log2) window around its reference key (scale 30), or are nearly flat
    (0.001): the end-of-pass check must route the first through the robust
    pass and both must stay within tolerance."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 6000, 8, 555)
    x.q = (x.q * scale).astype(np.float32)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


TREE32 = [-1] * 4 + [i // 4 - 1 for i in range(4, 32)]


@pytest.mark.parametrize("mode", [O.MODE_EXACT, O.MODE_APPROX])
def test_verify_c3_tree32_64k_refresh_then_reuse(oracle_lib, mode):
    """Config C3: 32-node draft tree at 64K context, a refresh layer and a
    reuse layer inheriting its index sets."""
    cfg = O.llama_config(32)
    x = LayerInputs(cfg, 65536, 32, 3232, parent_slot=TREE32)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, mode, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, mode, O.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)
    y = LayerInputs(cfg, 65536, 32, 3233, parent_slot=TREE32)
    case2 = DeviceCase(cfg, y)
    out2, _ = case2.run(4, mode, V.ROLE_REUSE, sets=sets)
    ref2 = case2.oracle(oracle_lib, 4, mode, O.ROLE_REUSE, idx=ref["idx"],
                        idx_count=ref["idx_count"], idx_forced=ref["idx_forced"])
    per, l2 = rel_errors(out2, ref2["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_c4_context_128k_chain8(oracle_lib):
    """Config C4's context length (131072 committed rows), one request, one layer."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 131072, 8, 12812)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


@pytest.mark.parametrize("gamma,mode,C", [(16, O.MODE_EXACT, 4), (16, O.MODE_APPROX, 4),
                                          (2, O.MODE_EXACT, 1)])
def test_verify_c5_draft_lengths(oracle_lib, gamma, mode, C):
    """Config C5's draft-length extremes (gamma 2 and 16 = routing lag) at 16K."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 16384, gamma, 1600 + gamma)
    case = DeviceCase(cfg, x)
    out, sets = case.run(C, mode, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, C, mode, O.ROLE_REFRESH)
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_batched_matches_per_request(oracle_lib):
    """specsv_nsa_verify_batched over three independent requests (different
    contexts, draft shapes and roles) sharing one workspace: every request's
    sets and outputs equal the per-request oracle's."""
    cfg = O.llama_config(4)
    specs = [(1000, 4, None, V.ROLE_REFRESH), (4096, 8, TREE8, V.ROLE_REFRESH),
             (3001, 2, None, V.ROLE_REUSE)]
    cases = [DeviceCase(cfg, LayerInputs(cfg, r, g, 500 + r, parent_slot=p)) for r, g, p, _ in specs]
    # the reuse request inherits sets built by a standalone refresh of the same request
    _, src_sets = cases[2].run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    src = sets_to_numpy(src_sets)
    sets = [V.IndexSets.empty(c.nq, cfg.n) for c in cases[:2]] + [src_sets]
    outs = [torch.zeros(c.nq, cfg.n_q_heads, cfg.d_head, device="cuda") for c in cases]
    # room for both REFRESH requests in one routing launch (the REUSE one routes nothing)
    ws = V.Workspace(cases[0].vcfg, max(c.nq for c in cases), max(c.x.k.shape[0] for c in cases),
                     batch=3)
    V.nsa_verify_batched(cases[0].vcfg, [c.cache for c in cases], [c.batch for c in cases], sets,
                         outs, ws, 4, V.MODE_EXACT, [s[3] for s in specs])
    torch.cuda.synchronize()
    for b, case in enumerate(cases):
        if specs[b][3] == V.ROLE_REFRESH:
            ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
            gi, gc, gf = sets_to_numpy(sets[b])
            assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
        else:
            ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REUSE, idx=src[0],
                              idx_count=src[1], idx_forced=forced_matrix(src[2], cfg.n))
        assert ref["rc"] == 0
        per, l2 = rel_errors(outs[b].cpu().numpy().astype(np.float64), ref["out"])
        assert per <= TOL and l2 <= TOL, (b, per, l2)


def test_verify_batched_validates_before_launch():
    """A bad request anywhere in the batch fails the call before any request's
    outputs are written."""
    cfg = O.llama_config(4)
    good = DeviceCase(cfg, LayerInputs(cfg, 2000, 2, 8))
    bad = DeviceCase(cfg, LayerInputs(cfg, 2000, 2, 9))
    bad.batch.pos = bad.batch.pos.copy()
    bad.batch.pos[2] = bad.batch.pos[0] + cfg.routing_lag + 1
    outs = [torch.full((3, cfg.n_q_heads, cfg.d_head), 7.0, device="cuda") for _ in range(2)]
    sets = [V.IndexSets.empty(3, cfg.n) for _ in range(2)]
    with pytest.raises(V.SpecsvError) as e:
        V.nsa_verify_batched(good.vcfg, [good.cache, bad.cache], [good.batch, bad.batch], sets,
                             outs, good.ws, 1, V.MODE_EXACT)
    assert e.value.code == 1
    torch.cuda.synchronize()
    assert bool((outs[0] == 7.0).all())


def test_c3_compressed_branch_repeated_fresh_caches(oracle_lib):
    """Regression: the attend kernel's per-tile P hand-off (p_full) once let a
    softmax warp running a tile ahead complete the previous tile's phase, so
    the PV MMA read another warp's P before it was written -- intermittently,
    mostly in the compressed branch of multi-chunk launches (33 queries = 3
    column chunks).  Repeated fresh runs with compressed-only gates; before
    the fix ~8% of runs failed (tools/stress_c3.py)."""
    cfg = O.llama_config(32)
    x = LayerInputs(cfg, 65536, 32, 3232, parent_slot=TREE32)
    x.gates = np.zeros_like(x.gates)
    x.gates[:, :, 0] = 1.0
    ref = None
    for _ in range(12):
        case = DeviceCase(cfg, x)
        out, _ = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
        if ref is None:
            ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)["out"]
        per, l2 = rel_errors(out, ref)
        assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_batched_many_requests_one_launch(oracle_lib):
    """10 requests (batched routing launches of 6 + 4, batched attend launches
    of 8 + 2 with fewer splits per head) against the same requests through
    single calls, and 3 against the oracle."""
    cfg = O.llama_config(4)
    specs = [(1000 + 350 * r, 4 if r % 2 else 8) for r in range(10)]
    cases = [DeviceCase(cfg, LayerInputs(cfg, rows, g, 700 + r)) for r, (rows, g) in enumerate(specs)]
    singles = [c.run(4, V.MODE_EXACT, V.ROLE_REFRESH) for c in cases]
    sets = [V.IndexSets.empty(c.nq, cfg.n) for c in cases]
    outs = [torch.zeros(c.nq, cfg.n_q_heads, cfg.d_head, device="cuda") for c in cases]
    # a workspace for 6 requests per routing launch: routing groups of 6 + 4
    ws = V.Workspace(cases[0].vcfg, max(c.nq for c in cases), max(c.x.k.shape[0] for c in cases),
                     batch=6)
    V.nsa_verify_batched(cases[0].vcfg, [c.cache for c in cases], [c.batch for c in cases], sets,
                         outs, ws, 4, V.MODE_EXACT)
    torch.cuda.synchronize()
    for r, case in enumerate(cases):
        s_out, s_sets = singles[r]
        gi, gc, gf = sets_to_numpy(sets[r])
        si, sc, sf = sets_to_numpy(s_sets)
        assert np.array_equal(gi, si) and np.array_equal(gc, sc) and np.array_equal(gf, sf)
        got = outs[r].cpu().numpy().astype(np.float64)
        assert np.abs(got - s_out).max() <= 1e-4 * max(np.abs(s_out).max(), 1e-6), r
        if r in (0, 5, 9):
            ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
            per, l2 = rel_errors(got, ref["out"])
            assert per <= TOL and l2 <= TOL, (r, per, l2)


def test_workspace_shared_across_query_counts(oracle_lib):
    """One workspace for calls with 33, 9 and 1 queries and a batched call:
    the attend barrier words sit at a fixed workspace offset, so a call never
    reads another call's partials as barrier words."""
    cfg = O.llama_config(4)
    vcfg = V.NsaConfig(**cfg.__dict__)
    ws = V.Workspace(vcfg, 65, 9000)
    for rows, g, parents in ((8192, 32, TREE32), (3000, 8, None), (2000, 0, None), (8192, 32, TREE32)):
        x = LayerInputs(cfg, rows, g, 60 + g + rows, parent_slot=parents)
        case = DeviceCase(cfg, x)
        case.ws = ws
        out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
        ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
        per, l2 = rel_errors(out, ref["out"])
        assert per <= TOL and l2 <= TOL, (rows, g, per, l2)


OTHER_CONFIGS = [
    # GQA group 2, wider window, more selected blocks, shorter lag
    dict(l=32, d=16, l_sel=64, n=24, w=1024, n_q_heads=8, n_kv_heads=4, d_head=128, routing_lag=8),
    # GQA group 8, fewer selected blocks, narrow window
    dict(l=32, d=16, l_sel=64, n=8, w=256, n_q_heads=16, n_kv_heads=2, d_head=128, routing_lag=16),
    # GQA group 16, longer compression blocks
    dict(l=64, d=16, l_sel=64, n=16, w=512, n_q_heads=16, n_kv_heads=1, d_head=128, routing_lag=16),
    # GQA group 32 (one query per column chunk)
    dict(l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=32, n_kv_heads=1, d_head=128, routing_lag=16),
    # n > 32: the Top-n selection's 8-lane groups (16-lane groups up to n = 32)
    dict(l=32, d=16, l_sel=64, n=48, w=512, n_q_heads=16, n_kv_heads=2, d_head=128, routing_lag=16),
]


@pytest.mark.parametrize("ci", range(len(OTHER_CONFIGS)))
@pytest.mark.parametrize("mode", [O.MODE_EXACT, O.MODE_APPROX])
def test_verify_other_nsa_configs(oracle_lib, ci, mode):
    """Configs beyond the Llama shape that this build accepts (GQA groups 2 to
    32, n, w, lag, l/d): indices and outputs against the oracle, refresh then
    reuse, on a tree draft."""
    cfg = O.NsaConfig(n_layers=4, **OTHER_CONFIGS[ci])
    x = LayerInputs(cfg, 5000, 8, 900 + ci, parent_slot=TREE8)
    case = DeviceCase(cfg, x)
    out, sets = case.run(2, mode, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 2, mode, O.ROLE_REFRESH)
    assert ref["rc"] == 0
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)
    y = LayerInputs(cfg, 5000, 8, 950 + ci, parent_slot=TREE8)
    case2 = DeviceCase(cfg, y)
    out2, _ = case2.run(2, mode, V.ROLE_REUSE, sets=sets)
    ref2 = case2.oracle(oracle_lib, 2, mode, O.ROLE_REUSE, idx=ref["idx"],
                        idx_count=ref["idx_count"], idx_forced=ref["idx_forced"])
    per, l2 = rel_errors(out2, ref2["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_config_beyond_build_limits_is_rejected():
    """A valid reference config this build does not cover (l=64, d=32: one
    16-block routing tile would touch more than 8 selection blocks) fails
    with EUNSUPPORTED before any launch, not with wrong results."""
    cfg = O.NsaConfig(n_layers=2, l=64, d=32, l_sel=64, n=16, w=512, n_q_heads=16, n_kv_heads=1,
                      d_head=128, routing_lag=16)
    x = LayerInputs(cfg, 3000, 2, 5)
    case = DeviceCase(cfg, x)
    with pytest.raises(V.SpecsvError) as e:
        case.run(1, V.MODE_EXACT, V.ROLE_REFRESH)
    assert e.value.code == 3


TREE64 = [-1] * 4 + [i // 4 - 1 for i in range(4, 64)]  # 64 nodes, depth <= 3


@pytest.mark.parametrize("mode", [O.MODE_EXACT, O.MODE_APPROX])
def test_verify_max_queries_tree64(oracle_lib, mode):
    """The largest call this build takes: 1 + 64 queries (six column chunks, a
    full 64-bit tree-mask word), refresh then reuse, against the oracle."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 8192, 64, 6464, parent_slot=TREE64)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, mode, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, mode, O.ROLE_REFRESH)
    assert ref["rc"] == 0
    gi, gc, gf = sets_to_numpy(sets)
    assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)
    y = LayerInputs(cfg, 8192, 64, 6465, parent_slot=TREE64)
    case2 = DeviceCase(cfg, y)
    out2, _ = case2.run(4, mode, V.ROLE_REUSE, sets=sets)
    ref2 = case2.oracle(oracle_lib, 4, mode, O.ROLE_REUSE, idx=ref["idx"],
                        idx_count=ref["idx_count"], idx_forced=ref["idx_forced"])
    per, l2 = rel_errors(out2, ref2["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_exact_grouping_equals_independent_queries(oracle_lib):
    """Exact coarsening is lossless (test_grouped_verifier.cpp:162-182): every
    draft query of a grouped call gets the indices and output it gets when it
    runs on its own.  On a chain, query i's independent execution is the call
    over the root and drafts 1..i (its ancestors; EXACT ownership keeps the
    other members out of its selected branch), a different launch (fewer
    columns, a smaller union, other tile-to-split assignment), so outputs agree
    up to fp32 summation order.  Query 0 (the root) also runs alone as a
    one-query call, and the grouped call matches the oracle at every C."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 6000, 8, 4321)
    case = DeviceCase(cfg, x)
    full, full_sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    fi, fc, ff = sets_to_numpy(full_sets)
    scale = max(np.abs(full).max(), 1e-6)
    b = case.batch
    for i in range(case.nq):
        sub = V.DraftBatch(pos=b.pos[:i + 1].copy(), tree_mask=x.tree_mask[:max(i, 1)].copy(),
                           q=b.q[:i + 1].contiguous(), gates=b.gates[:i + 1].contiguous(),
                           tree_k=b.tree_k[:i].contiguous() if i else None,
                           tree_v=b.tree_v[:i].contiguous() if i else None)
        sets = V.IndexSets.empty(i + 1, cfg.n)
        out = torch.zeros(i + 1, cfg.n_q_heads, cfg.d_head, device="cuda")
        V.nsa_verify(case.vcfg, case.cache, sub, sets, out, case.ws, 1, V.MODE_EXACT,
                     V.ROLE_REFRESH)
        torch.cuda.synchronize()
        si, sc, sf = sets_to_numpy(sets)
        assert sc[i] == fc[i] and np.array_equal(si[i], fi[i]) and sf[i] == ff[i], i
        got = out[i].cpu().numpy().astype(np.float64)
        assert np.abs(got - full[i]).max() <= 1e-5 * scale, i
    for C in (1, 2, 8):
        ref = case.oracle(oracle_lib, C, O.MODE_EXACT, O.ROLE_REFRESH)
        out, sets = case.run(C, V.MODE_EXACT, V.ROLE_REFRESH)
        gi, gc, gf = sets_to_numpy(sets)
        assert np.array_equal(gi, fi) and np.array_equal(gc, fc), C
        per, l2 = rel_errors(out, ref["out"])
        assert per <= TOL and l2 <= TOL, (C, per, l2)


ROUTE_VARIANTS = {"route3": {}, "route3_exact": {"SPECSV_ROUTE3_FORCE_EXACT": "1"},
                  "legacy": {"SPECSV_ROUTE_LEGACY": "1"}}


@pytest.mark.parametrize("rows,gamma,parents,mode", [(4096, 4, None, O.MODE_EXACT),
                                                     (3001, 8, TREE8, O.MODE_APPROX),
                                                     (65536, 8, None, O.MODE_EXACT)])
def test_route_kernels_agree(oracle_lib, monkeypatch, rows, gamma, parents, mode):
    """Routing runs on route3_kernel (integer tensor-pipe logits over the
    cache's digit planes, certified Top-n) by default;
    SPECSV_ROUTE3_FORCE_EXACT=1 sends every query through its exact fp64
    re-scoring path and SPECSV_ROUTE_LEGACY=1 selects the fp64-DMMA
    route_fused_kernel.  All three against the oracle, and their index sets
    agree; the fp64 score diagnostic holds P3."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, rows, gamma, 31 + rows + gamma, parent_slot=parents)
    case = DeviceCase(cfg, x)
    ref = case.oracle(oracle_lib, 4, mode, O.ROLE_REFRESH)
    got = {}
    for name, env in ROUTE_VARIANTS.items():
        for k in ("SPECSV_ROUTE3_FORCE_EXACT", "SPECSV_ROUTE_LEGACY"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out, sets = case.run(4, mode, V.ROLE_REFRESH)
        gi, gc, gf = sets_to_numpy(sets)
        assert _check_indices(oracle_lib, case, gi, gc, gf, ref) == 0, name
        per, l2 = rel_errors(out, ref["out"])
        assert per <= TOL and l2 <= TOL, (name, per, l2)
        got[name] = (gi, gc, gf)
    ck, _ = case.oracle_cache(oracle_lib)
    q = case.nq - 1
    sc = V.selection_scores(case.vcfg, case.cache, case.batch, q, case.ws).cpu().numpy()
    rs = oracle_lib.selection_scores(cfg, x.q[q], ck, cfg.routing_visible_len(int(x.pos[q])))
    assert np.abs(sc - rs).max() <= 1e-13 * np.abs(rs).max()
    for name in ROUTE_VARIANTS:
        for a, b in zip(got["route3"], got[name]):
            assert np.array_equal(a, b), name


def test_verify_batched_c4_shape(oracle_lib):
    """Config C4's own shape through the batched entry point: 16 requests at
    128K committed rows (gamma = 8 chain), ONE routing launch over all 16
    refresh requests and two attend launches of 8 (the per-GPU share of 64
    requests on 4 GPUs, what bench.py runs).  Every request's sets and outputs
    equal its single call; two requests are checked against the oracle; then a
    batched REUSE pass over the same sets equals the refresh outputs."""
    cfg = O.llama_config(4)
    vcfg = V.NsaConfig(**cfg.__dict__)
    R, rows, g = 16, 131072, 8
    nq = 1 + g
    oracle_reqs = {0: 31001, 11: 31011}
    cases = {r: DeviceCase(cfg, LayerInputs(cfg, rows, g, seed)) for r, seed in oracle_reqs.items()}
    gen = torch.Generator(device="cuda")
    caches, batches = [], []
    pos = np.array([rows - 1 + i for i in range(nq)], np.int64)
    from paper_2605_19893_b200.workload import chain_tree_mask
    for r in range(R):
        if r in cases:
            caches.append(cases[r].cache)
            batches.append(cases[r].batch)
            continue
        gen.manual_seed(7000 + r)
        c = V.LayerCache(vcfg, rows)
        u = lambda *s: torch.rand(*s, generator=gen, device="cuda") * 2 - 1  # noqa: E731
        c.append(u(rows, cfg.n_kv_heads, cfg.d_head).bfloat16(), u(rows, cfg.n_kv_heads, cfg.d_head).bfloat16())
        c.extend_compressed(u(cfg.l, cfg.d_head) * 0.1)
        caches.append(c)
        batches.append(V.DraftBatch(pos=pos.copy(), tree_mask=chain_tree_mask(g),
                                    q=u(nq, cfg.n_q_heads, cfg.d_head),
                                    gates=torch.rand(nq, cfg.n_q_heads, 3, generator=gen, device="cuda") * 0.6 + 0.2,
                                    tree_k=u(g, cfg.n_kv_heads, cfg.d_head).bfloat16(),
                                    tree_v=u(g, cfg.n_kv_heads, cfg.d_head).bfloat16()))
    ws1 = V.Workspace(vcfg, nq, rows)
    singles = []
    for r in range(R):
        s = V.IndexSets.empty(nq, cfg.n)
        o = torch.zeros(nq, cfg.n_q_heads, cfg.d_head, device="cuda")
        V.nsa_verify(vcfg, caches[r], batches[r], s, o, ws1, 4, V.MODE_EXACT, V.ROLE_REFRESH)
        singles.append((o, s))
    ws = V.Workspace(vcfg, nq, rows, batch=R)
    sets = [V.IndexSets.empty(nq, cfg.n) for _ in range(R)]
    outs = [torch.zeros(nq, cfg.n_q_heads, cfg.d_head, device="cuda") for _ in range(R)]
    V.nsa_verify_batched(vcfg, caches, batches, sets, outs, ws, 4, V.MODE_EXACT)
    outs2 = [torch.zeros_like(o) for o in outs]
    V.nsa_verify_batched(vcfg, caches, batches, sets, outs2, ws, 4, V.MODE_EXACT,
                         [V.ROLE_REUSE] * R)
    torch.cuda.synchronize()
    for r in range(R):
        so, ss = singles[r]
        gi, gc, gf = sets_to_numpy(sets[r])
        si, sc, sf = sets_to_numpy(ss)
        assert np.array_equal(gi, si) and np.array_equal(gc, sc) and np.array_equal(gf, sf), r
        got = outs[r].cpu().numpy().astype(np.float64)
        ref1 = so.cpu().numpy().astype(np.float64)
        assert np.abs(got - ref1).max() <= 1e-4 * max(np.abs(ref1).max(), 1e-6), r
        assert np.abs(outs2[r].cpu().numpy() - got).max() <= 1e-5 * max(np.abs(got).max(), 1e-6), r
        if r in cases:
            ref = cases[r].oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
            assert _check_indices(oracle_lib, cases[r], gi, gc, gf, ref) == 0, r
            per, l2 = rel_errors(got, ref["out"])
            assert per <= TOL and l2 <= TOL, (r, per, l2)
