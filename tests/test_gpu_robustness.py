"""GPU robustness of the C-ABI: KV-head-group shards, capacity bounds,
grids that cannot be co-resident, and verify calls racing other streams'
kernels.  All calls go through the C-ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200 import tree as T  # noqa: E402
from paper_2605_19893_b200 import verify as V  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402
from tests.gpu_harness import TOL, DeviceCase, rel_errors, sets_to_numpy  # noqa: E402

TREE8 = [-1, -1, 0, 0, 1, 2, 2, 4]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(case, C, mode, role, sets=None, kv_heads=None, fill=0.0):
    sets = sets or V.IndexSets.empty(case.nq, case.cfg.n)
    out = torch.full((case.nq, case.cfg.n_q_heads, case.cfg.d_head), fill, device="cuda")
    V.nsa_verify(case.vcfg, case.cache, case.batch, sets, out, case.ws, C, mode, role,
                 kv_heads=kv_heads)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), sets


@pytest.mark.parametrize("mode", [V.MODE_EXACT, V.MODE_APPROX])
def test_kv_head_shards_equal_the_full_call(mode):
    """KV-head group sharding (SURVEY 8e option i): every shard routes over all
    heads (same index sets as the full call), attends only its KV heads and
    writes only their q heads; the shards' union is the full call's output."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 7000, 8, 808, parent_slot=TREE8)
    case = DeviceCase(cfg, x)
    full, full_sets = _run(case, 4, mode, V.ROLE_REFRESH)
    fi, fc, ff = sets_to_numpy(full_sets)
    G = cfg.n_q_heads // cfg.n_kv_heads
    for shards in ([(0, 4), (4, 4)], [(0, 1), (1, 3), (4, 2), (6, 2)], [(h, 1) for h in range(8)]):
        merged = np.full_like(full, np.nan)
        for b, n in shards:
            out, sets = _run(case, 4, mode, V.ROLE_REFRESH, kv_heads=(b, n), fill=7.0)
            si, sc, sf = sets_to_numpy(sets)
            assert np.array_equal(si, fi) and np.array_equal(sc, fc) and np.array_equal(sf, ff)
            inside = slice(b * G, (b + n) * G)
            assert (out[:, :b * G] == 7.0).all() and (out[:, (b + n) * G:] == 7.0).all()
            merged[:, inside] = out[:, inside]
        assert not np.isnan(merged).any()
        assert np.abs(merged - full).max() <= 1e-5 * max(np.abs(full).max(), 1e-6), shards
    # reuse layers shard the same way (no routing at all)
    y = LayerInputs(cfg, 7000, 8, 809, parent_slot=TREE8)
    case2 = DeviceCase(cfg, y)
    full2, _ = _run(case2, 4, mode, V.ROLE_REUSE, sets=full_sets)
    for b, n in [(0, 4), (4, 4)]:
        out, _ = _run(case2, 4, mode, V.ROLE_REUSE, sets=full_sets, kv_heads=(b, n), fill=7.0)
        inside = slice(b * G, (b + n) * G)
        assert np.abs(out[:, inside] - full2[:, inside]).max() <= 1e-5 * max(np.abs(full2).max(), 1e-6)


def test_kv_head_range_rejected_outside_the_config():
    cfg = O.llama_config(4)
    case = DeviceCase(cfg, LayerInputs(cfg, 2000, 2, 5))
    for bad in ((7, 2), (-1, 1), (3, -1), (2, 0)):
        with pytest.raises(V.SpecsvError) as e:
            _run(case, 1, V.MODE_EXACT, V.ROLE_REFRESH, kv_heads=bad)
        assert e.value.code == 1, bad


def test_batched_kv_head_shards(oracle_lib):
    """The batched entry point with a KV-head range per request."""
    cfg = O.llama_config(4)
    cases = [DeviceCase(cfg, LayerInputs(cfg, 3000 + 500 * r, 8, 40 + r)) for r in range(3)]
    fulls = [c.run(4, V.MODE_EXACT, V.ROLE_REFRESH)[0] for c in cases]
    heads = [(0, 4), (4, 4), (2, 3)]
    G = cfg.n_q_heads // cfg.n_kv_heads
    sets = [V.IndexSets.empty(c.nq, cfg.n) for c in cases]
    outs = [torch.full((c.nq, cfg.n_q_heads, cfg.d_head), 7.0, device="cuda") for c in cases]
    ws = V.Workspace(cases[0].vcfg, 9, 4000, batch=3)
    V.nsa_verify_batched(cases[0].vcfg, [c.cache for c in cases], [c.batch for c in cases], sets,
                         outs, ws, 4, V.MODE_EXACT, kv_heads=heads)
    torch.cuda.synchronize()
    for r, (b, n) in enumerate(heads):
        got = outs[r].cpu().numpy().astype(np.float64)
        inside = slice(b * G, (b + n) * G)
        assert np.abs(got[:, inside] - fulls[r][:, inside]).max() <= 1e-4 * np.abs(fulls[r]).max()
        assert (got[:, :b * G] == 7.0).all() and (got[:, (b + n) * G:] == 7.0).all()


def test_rows_beyond_capacity_rejected():
    cfg = O.llama_config(4)
    case = DeviceCase(cfg, LayerInputs(cfg, 2000, 2, 11))
    case.cache.rows = case.cache.capacity + 1
    with pytest.raises(V.SpecsvError) as e:
        case.run(1, V.MODE_EXACT, V.ROLE_REFRESH)
    assert e.value.code == 1


def test_commit_beyond_capacity_rejected_by_the_library():
    """specsv_commit_rows bounds-checks rows + n_accepted against the cache
    capacity itself (the Python check is bypassed here)."""
    import ctypes as C
    from paper_2605_19893_b200 import abi
    cfg = V.NsaConfig(n_layers=1)
    cache = V.LayerCache(cfg, 100)
    cache.rows = 98
    tk = torch.zeros(4, cfg.n_kv_heads, cfg.d_head, dtype=torch.bfloat16, device="cuda")
    slots = np.array([0, 1, 2], np.int32)
    kvs = (abi.LayerKvC * 1)(cache.c())
    ptrs = (C.c_void_p * 1)(tk.data_ptr())
    c = cfg.c()
    rc = T._lib().specsv_commit_rows(C.byref(c), kvs, ptrs, ptrs, 1,
                                     slots.ctypes.data_as(C.POINTER(C.c_int32)), 3, None)
    assert rc == 1
    assert b"capacity" in abi.lib().specsv_last_error()


def test_many_heads_single_split_launch(oracle_lib):
    """Hq=128 / Hkv=16 with 1 + 64 queries: 11 column chunks x 16 KV heads =
    176 CTA groups, more than the co-resident CTAs, so the attend launch runs
    one split per head, non-cooperatively, in several waves (it used to be
    launched cooperatively and fail)."""
    cfg = O.NsaConfig(n_layers=2, l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=128,
                      n_kv_heads=16, d_head=128, routing_lag=16)
    parents = [-1] * 4 + [i // 4 - 1 for i in range(4, 64)]
    x = LayerInputs(cfg, 2500, 64, 4096, parent_slot=parents)
    case = DeviceCase(cfg, x)
    out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    ref = case.oracle(oracle_lib, 4, O.MODE_EXACT, O.ROLE_REFRESH)
    assert ref["rc"] == 0
    gi, gc, _ = sets_to_numpy(sets)
    for q in range(case.nq):
        assert gc[q] == ref["idx_count"][q] and (gi[q, :gc[q]] == ref["idx"][q, :gc[q]]).all(), q
    per, l2 = rel_errors(out, ref["out"])
    assert per <= TOL and l2 <= TOL, (per, l2)


def test_verify_while_other_streams_occupy_the_sms(oracle_lib):
    """The routing and attend launches are cooperative (all CTAs co-resident);
    with long GEMMs running on another stream at the same time, the driver
    must still place the whole grid and the results must not change."""
    cfg = O.llama_config(4)
    x = LayerInputs(cfg, 9000, 8, 99)
    case = DeviceCase(cfg, x)
    want, want_sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for _ in range(20):
            a = (a @ a).clamp_(-1, 1)
    for _ in range(5):
        out, sets = case.run(4, V.MODE_EXACT, V.ROLE_REFRESH)
        assert np.array_equal(out, want)
        assert torch.equal(sets.idx, want_sets.idx)
    side.synchronize()
