"""ctypes/numpy front end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two libraries export the same C API (``oracle/nsa_oracle.h``):

* ``oracle/liboracle.so``          -- the plain-C restatement (always built);
* ``oracle/_ref/libspecsv_ref.so`` -- the reference itself compiled in place
  from /root/reference/proj/src plus ``ref_shim.cpp`` (built where the
  reference is mounted; the built .so travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecsv_ref.so")

MODE_EXACT, MODE_APPROX = 0, 1
ROLE_REFRESH, ROLE_REUSE = 0, 1


class OrConfig(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("l", "d", "l_sel", "n", "w", "n_q_heads", "n_kv_heads", "d_head",
                 "n_layers", "routing_lag")]


OR_MAX_PAIRS = 128


class OrStats(C.Structure):
    _fields_ = [("unique_block_loads", C.c_int64), ("total_requested_loads", C.c_int64),
                ("dedup_savings", C.c_int64), ("window_token_loads", C.c_int64),
                ("launches", C.c_int64), ("index_constructions", C.c_int64),
                ("n_pairs", C.c_int64), ("pairwise_overlap", C.c_int64 * OR_MAX_PAIRS)]

    def as_dict(self):
        return {
            "unique_block_loads": self.unique_block_loads,
            "total_requested_loads": self.total_requested_loads,
            "dedup_savings": self.dedup_savings,
            "window_token_loads": self.window_token_loads,
            "launches": self.launches,
            "index_constructions": self.index_constructions,
            "pairwise_overlap": [self.pairwise_overlap[i] for i in range(self.n_pairs)],
        }


@dataclass
class NsaConfig:
    """Mirror of ``NsaConfig`` (include/specsv/nsa/config.hpp:24-34)."""
    l: int = 32
    d: int = 16
    l_sel: int = 64
    n: int = 16
    w: int = 512
    n_q_heads: int = 4
    n_kv_heads: int = 2
    d_head: int = 64
    n_layers: int = 8
    routing_lag: int = 16

    def c(self) -> OrConfig:
        return OrConfig(self.l, self.d, self.l_sel, self.n, self.w, self.n_q_heads,
                        self.n_kv_heads, self.d_head, self.n_layers, self.routing_lag)

    def routing_visible_len(self, pos: int) -> int:
        return max(0, pos + 1 - self.routing_lag)


def small_config() -> NsaConfig:
    """tests/test_util.hpp:16-29."""
    return NsaConfig(l=8, d=4, l_sel=16, n=4, w=32, n_q_heads=2, n_kv_heads=1, d_head=8,
                     n_layers=2, routing_lag=8)


def llama_config(n_layers: int = 32) -> NsaConfig:
    """Llama-3.1-8B-shaped NSA (BASELINE.json configs)."""
    return NsaConfig(l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=32, n_kv_heads=8,
                     d_head=128, n_layers=n_layers, routing_lag=16)


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path}")
        self.path = path
        L = self.lib = C.CDLL(path)
        i64, u64, f32p, f64p = C.c_int64, C.c_uint64, C.POINTER(C.c_float), C.POINTER(C.c_double)
        i64p, u8p, i32p, u64p = (C.POINTER(C.c_int64), C.POINTER(C.c_uint8),
                                 C.POINTER(C.c_int32), C.POINTER(C.c_uint64))
        cfgp = C.POINTER(OrConfig)
        L.or_impl_name.restype = C.c_char_p
        L.or_validate.argtypes = [cfgp]
        L.or_rng_fill_symmetric.argtypes = [u64, C.c_float, f32p, i64]
        L.or_rng_fill_symmetric.restype = u64
        L.or_dot_f32.argtypes = [f32p, f32p, i64]
        L.or_dot_f32.restype = C.c_double
        L.or_compressed_block_count.argtypes = [i64, cfgp]
        L.or_compressed_block_count.restype = i64
        L.or_build_compressed.argtypes = [cfgp, f32p, f32p, i64, f32p, f32p, f32p]
        L.or_build_compressed.restype = i64
        L.or_selection_scores.argtypes = [cfgp, f32p, f32p, i64, i64, f64p]
        L.or_selection_scores.restype = i64
        L.or_select_blocks.argtypes = [cfgp, f64p, i64, i64, i64p, i64, i64p, u8p]
        L.or_select_blocks.restype = i64
        L.or_branch_compressed.argtypes = [cfgp, f32p, f32p, f32p, i64, i64, f64p]
        L.or_branch_selected.argtypes = [cfgp, f32p, f32p, f32p, i64, i64p, i64, u8p, i64, f64p]
        L.or_branch_window.argtypes = [cfgp, f32p, f32p, f32p, i64, i64, i64, f32p, f32p, i32p,
                                       i64, f64p]
        L.or_merge_partials.argtypes = [i64, f64p, f64p, f64p]
        L.or_gated_combine.argtypes = [i64, f64p, f64p, f64p, f64p, f64p]
        L.or_merged_schedule.argtypes = [i64p, i64p, i64, i64, i64p, u8p]
        L.or_merged_schedule.restype = i64
        L.or_representative_index.argtypes = [i64p, i64]
        L.or_representative_index.restype = i64
        L.or_clamp_inherited.argtypes = [cfgp, i64p, u8p, i64, i64, i64p, u8p]
        L.or_clamp_inherited.restype = i64
        L.or_verify_layer.argtypes = [cfgp, f32p, f32p, i64, f32p, f32p, i64, f32p, f32p, i64,
                                      f32p, i64p, f64p, u64p, i64, i64, C.c_int, C.c_int, i64p,
                                      i64p, u8p, f64p, C.POINTER(OrStats)]

    @property
    def name(self) -> str:
        return self.lib.or_impl_name().decode()

    # -- thin wrappers -------------------------------------------------------
    def validate(self, cfg: NsaConfig) -> bool:
        c = cfg.c()
        return self.lib.or_validate(C.byref(c)) == 0

    def rng_symmetric(self, seed: int, a: float, count: int):
        out = np.empty(count, np.float32)
        st = self.lib.or_rng_fill_symmetric(seed, a, _p(out, C.c_float), count)
        return out, st

    def dot(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.or_dot_f32(_p(a, C.c_float), _p(b, C.c_float), a.size)

    def compressed_block_count(self, rows: int, cfg: NsaConfig) -> int:
        c = cfg.c()
        return self.lib.or_compressed_block_count(rows, C.byref(c))

    def build_compressed(self, cfg, k, v, committed_len, pe=None):
        c = cfg.c()
        nb = max(0, self.compressed_block_count(committed_len, cfg))
        ck = np.zeros((max(nb, 1), cfg.n_kv_heads, cfg.d_head), np.float32)
        cv = np.zeros_like(ck)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        pe = None if pe is None else np.ascontiguousarray(pe, np.float32)
        got = self.lib.or_build_compressed(C.byref(c), _p(k, C.c_float), _p(v, C.c_float),
                                           committed_len, _p(pe, C.c_float),
                                           _p(ck, C.c_float), _p(cv, C.c_float))
        return ck[:got], cv[:got]

    def selection_scores(self, cfg, q, ck, visible_len):
        c = cfg.c()
        q = np.ascontiguousarray(q, np.float32)
        ck = np.ascontiguousarray(ck, np.float32)
        out = np.zeros(max(1, -(-visible_len // cfg.l_sel)), np.float64)
        n = self.lib.or_selection_scores(C.byref(c), _p(q, C.c_float), _p(ck, C.c_float),
                                         ck.shape[0], visible_len, _p(out, C.c_double))
        return out[:n]

    def select_blocks(self, cfg, scores, n, visible_len, forced=None):
        c = cfg.c()
        scores = np.ascontiguousarray(scores, np.float64)
        idx = np.zeros(max(1, n + 3), np.int64)
        fl = np.zeros(max(1, n + 3), np.uint8)
        fa = None if forced is None else np.ascontiguousarray(forced, np.int64)
        cnt = self.lib.or_select_blocks(C.byref(c), _p(scores, C.c_double), n, visible_len,
                                        _p(fa, C.c_int64), 0 if fa is None else fa.size,
                                        _p(idx, C.c_int64), _p(fl, C.c_uint8))
        return idx[:cnt].tolist(), [bool(x) for x in fl[:cnt]]

    def merged_schedule(self, sets):
        stride = max([len(s) for s in sets] + [1])
        arr = np.full((len(sets), stride), -1, np.int64)
        for i, s in enumerate(sets):
            arr[i, :len(s)] = s
        counts = np.array([len(s) for s in sets], np.int64)
        uniq = np.zeros(max(1, arr.size), np.int64)
        own = np.zeros(max(1, arr.size * len(sets)), np.uint8)
        nu = self.lib.or_merged_schedule(_p(arr, C.c_int64), _p(counts, C.c_int64), len(sets),
                                         stride, _p(uniq, C.c_int64), _p(own, C.c_uint8))
        own = own[: nu * len(sets)].reshape(len(sets), nu).astype(bool)
        return uniq[:nu].tolist(), own.tolist()

    def representative_index(self, positions):
        p = np.ascontiguousarray(positions, np.int64)
        return self.lib.or_representative_index(_p(p, C.c_int64), p.size)

    def clamp_inherited(self, cfg, src, forced, bound):
        c = cfg.c()
        s = np.ascontiguousarray(src, np.int64)
        f = np.ascontiguousarray(forced, np.uint8)
        out = np.zeros(max(1, s.size), np.int64)
        of = np.zeros(max(1, s.size), np.uint8)
        n = self.lib.or_clamp_inherited(C.byref(c), _p(s, C.c_int64), _p(f, C.c_uint8), s.size,
                                        bound, _p(out, C.c_int64), _p(of, C.c_uint8))
        return out[:n].tolist(), [bool(x) for x in of[:n]]

    def branch_compressed(self, cfg, q, ck, cv, visible_len):
        c = cfg.c()
        out = np.zeros((cfg.n_q_heads, cfg.d_head + 2), np.float64)
        q, ck, cv = (np.ascontiguousarray(x, np.float32) for x in (q, ck, cv))
        self.lib.or_branch_compressed(C.byref(c), _p(q, C.c_float), _p(ck, C.c_float),
                                      _p(cv, C.c_float), ck.shape[0], visible_len,
                                      _p(out, C.c_double))
        return out

    def branch_selected(self, cfg, q, k, v, blocks, token_bound, ownership=None):
        c = cfg.c()
        out = np.zeros((cfg.n_q_heads, cfg.d_head + 2), np.float64)
        q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
        b = np.ascontiguousarray(blocks, np.int64)
        own = None if ownership is None else np.ascontiguousarray(ownership, np.uint8)
        self.lib.or_branch_selected(C.byref(c), _p(q, C.c_float), _p(k, C.c_float),
                                    _p(v, C.c_float), k.shape[0], _p(b, C.c_int64), b.size,
                                    _p(own, C.c_uint8), token_bound, _p(out, C.c_double))
        return out

    def branch_window(self, cfg, q, k, v, pos, committed_len, tree_k=None, tree_v=None,
                      admitted=()):
        c = cfg.c()
        out = np.zeros((cfg.n_q_heads, cfg.d_head + 2), np.float64)
        q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
        tk = None if tree_k is None else np.ascontiguousarray(tree_k, np.float32)
        tv = None if tree_v is None else np.ascontiguousarray(tree_v, np.float32)
        adm = np.ascontiguousarray(admitted, np.int32)
        self.lib.or_branch_window(C.byref(c), _p(q, C.c_float), _p(k, C.c_float),
                                  _p(v, C.c_float), k.shape[0], pos, committed_len,
                                  _p(tk, C.c_float), _p(tv, C.c_float), _p(adm, C.c_int32),
                                  adm.size, _p(out, C.c_double))
        return out

    def merge_partials(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        r = np.zeros_like(a)
        self.lib.or_merge_partials(a.size - 2, _p(a, C.c_double), _p(b, C.c_double),
                                   _p(r, C.c_double))
        return r

    def gated_combine(self, cmp, slc, win, gates):
        cmp, slc, win = (np.ascontiguousarray(x, np.float64) for x in (cmp, slc, win))
        g = np.ascontiguousarray(gates, np.float64)
        out = np.zeros(cmp.size - 2, np.float64)
        self.lib.or_gated_combine(cmp.size - 2, _p(cmp, C.c_double), _p(slc, C.c_double),
                                  _p(win, C.c_double), _p(g, C.c_double), _p(out, C.c_double))
        return out

    def verify_layer(self, cfg, k, v, ck, cv, q, pos, gates, tree_k=None, tree_v=None,
                     tree_mask=None, group_size=4, mode=MODE_EXACT, role=ROLE_REFRESH,
                     idx=None, idx_count=None, idx_forced=None):
        """Per-layer verify (engine.cpp:175-278).  Returns dict with out [nq][Hq][dh]
        (fp64), idx [nq][n], idx_count [nq], idx_forced [nq][n], stats, rc."""
        c = cfg.c()
        k, v, ck, cv, q = (np.ascontiguousarray(x, np.float32) for x in (k, v, ck, cv, q))
        nq = q.shape[0]
        gamma = nq - 1
        pos = np.ascontiguousarray(pos, np.int64)
        gates = np.ascontiguousarray(gates, np.float64)
        words = max(1, (gamma + 63) // 64)
        if tree_mask is None:
            tree_mask = np.zeros((max(gamma, 1), words), np.uint64)
        tree_mask = np.ascontiguousarray(tree_mask, np.uint64)
        if gamma > 0:
            tk = np.ascontiguousarray(tree_k, np.float32)
            tv = np.ascontiguousarray(tree_v, np.float32)
        else:
            tk = tv = None
        n = cfg.n
        idx = np.full((nq, n), -1, np.int64) if idx is None else np.array(idx, np.int64)
        cnt = (np.full(nq, -1, np.int64) if idx_count is None
               else np.array(idx_count, np.int64))
        fl = np.zeros((nq, n), np.uint8) if idx_forced is None else np.array(idx_forced, np.uint8)
        out = np.zeros((nq, cfg.n_q_heads, cfg.d_head), np.float64)
        st = OrStats()
        rc = self.lib.or_verify_layer(C.byref(c), _p(k, C.c_float), _p(v, C.c_float), k.shape[0],
                                      _p(ck, C.c_float), _p(cv, C.c_float), ck.shape[0],
                                      _p(tk, C.c_float), _p(tv, C.c_float), nq, _p(q, C.c_float),
                                      _p(pos, C.c_int64), _p(gates, C.c_double),
                                      _p(tree_mask, C.c_uint64), words, group_size, mode, role,
                                      _p(idx, C.c_int64), _p(cnt, C.c_int64), _p(fl, C.c_uint8),
                                      _p(out, C.c_double), C.byref(st))
        return {"rc": rc, "out": out, "idx": idx, "idx_count": cnt, "idx_forced": fl,
                "stats": st.as_dict()}


def load(which: str = "oracle") -> Oracle:
    return Oracle(REF_SO if which == "ref" else ORACLE_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefTree:
    """The reference's own draft-tree utilities (proj/src/draft_tree.cpp) via
    oracle/ref_tree_shim.cpp in oracle/_ref -- the checker for
    include/specsv_b200/draft_tree.h.  Trees are flat arrays (node 0 root)."""

    PROPOSE = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                          C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_double))

    def __init__(self, path: str = REF_SO):
        self.L = C.CDLL(path)

    def expand(self, root_token, propose, D, k, budget=None, capacity=4096):
        """propose(node_id, token, depth, cum_score, k) -> [(token, score), ...]"""
        arrs = (np.zeros(capacity, np.int64), np.zeros(capacity, np.int32),
                np.zeros(capacity, np.int32), np.zeros(capacity, np.float64),
                np.zeros(capacity, np.float64))

        def cb(_ctx, node, tok, dep, cs, kk, tout, sout):
            top = list(propose(int(node), int(tok), int(dep), float(cs), int(kk)))
            for i, (t, s) in enumerate(top):
                tout[i] = int(t)
                sout[i] = float(s)
            return len(top)

        n = C.c_int64(0)
        rc = self.L.or_ref_tree_expand(C.c_int32(root_token), self.PROPOSE(cb), None, C.c_int64(D),
                                       C.c_int64(k), C.c_int64(-1 if budget is None else budget),
                                       C.c_int64(capacity), _p(arrs[0], C.c_int64),
                                       _p(arrs[1], C.c_int32), _p(arrs[2], C.c_int32),
                                       _p(arrs[3], C.c_double), _p(arrs[4], C.c_double),
                                       C.byref(n))
        m = n.value
        return rc, tuple(a[:m].copy() for a in arrs)

    def flatten(self, parent, token, depth, score, traversal, committed_len):
        n = len(parent)
        g = n - 1
        arrs = [np.ascontiguousarray(parent, np.int64), np.ascontiguousarray(token, np.int32),
                np.ascontiguousarray(depth, np.int32), np.ascontiguousarray(score, np.float64)]
        order = np.zeros(max(g, 1), np.int64)
        pos = np.zeros(max(g, 1), np.int64)
        mask = np.zeros((max(g, 1), max(g, 1)), np.uint8)
        self.L.or_ref_tree_flatten(C.c_int64(n), _p(arrs[0], C.c_int64), _p(arrs[1], C.c_int32),
                                   _p(arrs[2], C.c_int32), _p(arrs[3], C.c_double),
                                   C.c_int32(traversal), C.c_int64(committed_len),
                                   _p(order, C.c_int64), _p(pos, C.c_int64), _p(mask, C.c_uint8))
        return order[:g], pos[:g], mask[:g, :g].astype(bool)

    def greedy(self, parent, token, depth, score, argmax):
        n = len(parent)
        arrs = [np.ascontiguousarray(parent, np.int64), np.ascontiguousarray(token, np.int32),
                np.ascontiguousarray(depth, np.int32), np.ascontiguousarray(score, np.float64),
                np.ascontiguousarray(argmax, np.int32)]
        nodes = np.zeros(max(n, 1), np.int64)
        toks = np.zeros(max(n, 1), np.int32)
        na, bonus = C.c_int64(0), C.c_int32(0)
        rc = self.L.or_ref_tree_greedy(C.c_int64(n), _p(arrs[0], C.c_int64), _p(arrs[1], C.c_int32),
                                       _p(arrs[2], C.c_int32), _p(arrs[3], C.c_double),
                                       _p(arrs[4], C.c_int32), _p(nodes, C.c_int64),
                                       _p(toks, C.c_int32), C.byref(na), C.byref(bonus))
        return rc, nodes[:na.value].tolist(), toks[:na.value].tolist(), int(bonus.value)
