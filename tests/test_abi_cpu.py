"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host policy (validation, layer roles, clamping,
LoadStats) follows the reference rules.  No device compute here."""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_19893_b200 import abi
from paper_2605_19893_b200 import verify as V
from paper_2605_19893_b200.workload import LayerInputs

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "specsv_b200",
                      "nsa_verify.h")


def test_library_exports_every_declared_symbol():
    decl = set(re.findall(r"\b(specsv_[a-z_0-9]+)\s*\(", open(HEADER).read()))
    assert decl == set(abi.EXPORTED)
    L = abi.lib()
    for name in decl:
        assert hasattr(L, name), name
    assert L.specsv_abi_version() == 3


def test_validate_config_rules():
    V.NsaConfig().validate()
    for field, val in (("d", 33), ("l_sel", 17), ("n", 2), ("n_q_heads", 31), ("w", 8)):
        bad = V.NsaConfig(**{**V.NsaConfig().__dict__, field: val})
        with pytest.raises(abi.SpecsvError) as e:
            bad.validate()
        assert e.value.code == abi.EINVAL
    with pytest.raises(abi.SpecsvError) as e:
        V.NsaConfig(d_head=64).validate()
    assert e.value.code == abi.EUNSUPPORTED


def test_resolve_layer_roles_kats():  # test_fusion_schedule.cpp:11-50
    S = [3, 6, 7, 8, 12, 13, 14, 15]
    roles, src = V.resolve_layer_roles(S, 16)
    assert src[3] == 2 and src[6] == 5 and src[7] == 5 and src[8] == 5
    assert all(src[j] == 11 for j in (12, 13, 14, 15))
    assert all(src[j] == j for j in range(16) if roles[j] == V.ROLE_REFRESH)
    assert (roles == V.ROLE_REFRESH).sum() == 8
    alt = list(range(1, 16, 2))
    roles, src = V.resolve_layer_roles(alt, 16)
    assert all(src[j] == j - 1 for j in alt)
    for bad in ([0], [8], [-1]):
        with pytest.raises(abi.SpecsvError):
            V.resolve_layer_roles(bad, 8)


def test_clamp_kats():  # test_fusion_schedule.cpp:56-80
    cfg = V.NsaConfig()
    src, fb = [0, 2, 5, 9], 0b1001
    assert V.clamp_inherited_indices(cfg, src, fb, 10 * 64) == (src, [True, False, False, True])
    assert V.clamp_inherited_indices(cfg, src, fb, 5 * 64 + 10)[0] == [0, 2, 5]
    assert V.clamp_inherited_indices(cfg, src, fb, 64) == ([0], [True])


@pytest.mark.parametrize("mode", [O.MODE_EXACT, O.MODE_APPROX])
@pytest.mark.parametrize("C", [1, 2, 4])
@pytest.mark.parametrize("tree", [False, True])
def test_load_stats_match_reference(oracle_lib, mode, C, tree):
    cfg = O.llama_config(4)
    parents = [-1, -1, 0, 0, 1, 2, 2, 4] if tree else None
    x = LayerInputs(cfg, 1500, 8, 11 + C, parent_slot=parents)
    ck, cv = oracle_lib.build_compressed(cfg, x.k, x.v, x.k.shape[0], x.pos_embed)
    vcfg = V.NsaConfig(**cfg.__dict__)
    for role in (O.ROLE_REFRESH, O.ROLE_REUSE):
        kw = {}
        if role == O.ROLE_REUSE:
            kw = dict(idx=prev["idx"], idx_count=prev["idx_count"], idx_forced=prev["idx_forced"])
        r = oracle_lib.verify_layer(cfg, x.k, x.v, ck, cv, x.q, x.pos, x.gates.astype(np.float64),
                                    x.tree_k, x.tree_v, x.tree_mask, C, mode, role, **kw)
        prev = r
        got = V.load_stats(vcfg, x.k.shape[0], x.pos, x.tree_mask, r["idx"].astype(np.int32),
                           r["idx_count"].astype(np.int32), C, mode, role)
        assert got == r["stats"]


def test_algorithmic_bytes_counts_union_once():
    cfg = V.NsaConfig()
    rows = 65536
    pos = np.array([rows - 1 + i for i in range(9)], np.int64)
    idx = np.full((9, 16), -1, np.int32)
    cnt = np.full(9, 16, np.int32)
    base = [0] + list(range(10, 23)) + [1022, 1023]
    for q in range(9):
        idx[q] = sorted(base)
    b = V.algorithmic_bytes(cfg, rows, pos, V.ROLE_REUSE, idx, cnt, V.MODE_EXACT, 4)
    m = (rows - 16 - 32) // 16 + 1
    tokens = 14 * 64 + 512  # 14 distinct non-window blocks + the window (covers 1022, 1023)
    expect = m * 8 * 128 * 4 + tokens * 8 * 128 * 4 + 8 * 8 * 128 * 4 + 9 * 32 * 128 * 8 + 9 * 32 * 12
    assert b == expect


def test_workspace_sizes():
    """The single-request workspace covers every query count up to 65 at its
    row bound; the batched size adds one routing region per extra REFRESH
    request up to the 16 a routing launch takes, and no more."""
    import ctypes as C
    L = abi.lib()
    c = V.NsaConfig(l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=32, n_kv_heads=8, d_head=128,
                    n_layers=32, routing_lag=16).c()
    one = L.specsv_verify_workspace_size(C.byref(c), 9, 65536)
    assert one > 0
    assert L.specsv_verify_workspace_size(C.byref(c), 65, 65536) >= one
    assert L.specsv_verify_workspace_size(C.byref(c), 9, 131072) > one
    assert L.specsv_verify_workspace_size_batched(C.byref(c), 9, 65536, 1) == one
    sizes = [L.specsv_verify_workspace_size_batched(C.byref(c), 9, 65536, b) for b in (2, 8, 16, 17, 64)]
    step = sizes[0] - one
    assert step > 0
    assert sizes[1] == one + 7 * step and sizes[2] == one + 15 * step
    assert sizes[3] == sizes[2] and sizes[4] == sizes[2]  # a routing launch takes at most 16
    assert L.specsv_verify_workspace_size_batched(C.byref(c), 9, 65536, 0) == 0
