"""Python face of the B200 verify path, mirroring the reference operator API.

Reference names (paths relative to /root/reference/proj):
  NsaConfig           include/specsv/nsa/config.hpp:24-59
  LayerCache          LayerKv + CompressedLayer, include/specsv/nsa/cache.hpp:15-82
  LayerCache.extend_compressed   nsa::extend_compressed_layer (cache.hpp:91-97)
  nsa_verify          per-layer section of run_target_pass (src/engine.cpp:175-278)
  route               nsa::selection_scores + select_blocks (nsa/attention.hpp:29-44)
  attend_fused        verify::group_attend_exact/approx (verify/group_attend.hpp:50-66)
  resolve_layer_roles / clamp_inherited_indices  schedule/layer_roles.hpp:45-57
  load_stats          verify::LoadStats (verify/grouping.hpp:33-52)

Device memory comes from torch (plumbing); every computation runs in the
sm_100a library through the C-ABI.  Errors raise SpecsvError with the same
conditions under which the reference throws std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import abi
from .abi import MODE_APPROX, MODE_EXACT, ROLE_REFRESH, ROLE_REUSE, SpecsvError, check, lib

__all__ = ["NsaConfig", "LayerCache", "IndexSets", "DraftBatch", "Workspace", "nsa_verify",
           "nsa_verify_batched", "PreparedVerify",
           "route", "attend_fused", "selection_scores", "select_blocks", "resolve_layer_roles",
           "clamp_inherited_indices", "load_stats", "algorithmic_bytes", "MODE_EXACT",
           "MODE_APPROX", "ROLE_REFRESH", "ROLE_REUSE", "SpecsvError"]


@dataclass
class NsaConfig:
    l: int = 32
    d: int = 16
    l_sel: int = 64
    n: int = 16
    w: int = 512
    n_q_heads: int = 32
    n_kv_heads: int = 8
    d_head: int = 128
    n_layers: int = 32
    routing_lag: int = 16

    def c(self) -> abi.NsaConfigC:
        return abi.NsaConfigC(self.l, self.d, self.l_sel, self.n, self.w, self.n_q_heads,
                              self.n_kv_heads, self.d_head, self.n_layers, self.routing_lag)

    def validate(self) -> None:
        c = self.c()
        check(lib().specsv_validate_config(C.byref(c)))

    @property
    def gqa_group_size(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    def routing_visible_len(self, pos: int) -> int:
        return max(0, pos + 1 - self.routing_lag)

    def compressed_block_count(self, rows: int) -> int:
        return (rows - self.l) // self.d + 1 if rows >= self.l else 0


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class LayerCache:
    """Device-resident committed K/V (bf16, [row][kv_head][d_head]) plus the
    compressed cache (fp32 routing keys, bf16 key copy, bf16 pooled values)."""

    def __init__(self, cfg: NsaConfig, capacity: int, device="cuda"):
        self.cfg = cfg
        H, dh = cfg.n_kv_heads, cfg.d_head
        self.capacity = capacity
        self.k = torch.zeros(capacity, H, dh, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros_like(self.k)
        nb = max(1, cfg.compressed_block_count(capacity))
        self.ck = torch.zeros(nb, H, dh, dtype=torch.float32, device=device)
        self.ck16 = torch.zeros(nb, H, dh, dtype=torch.bfloat16, device=device)
        self.cv = torch.zeros_like(self.ck16)
        # routing keys as fixed-point digit planes (int8 [blocks][Hkv][4][dh])
        # and their row exponents, written with ck by every compressed append
        self.ckd = torch.zeros(nb, H, 4, dh, dtype=torch.int8, device=device)
        self.ckexp = torch.zeros(nb, H, dtype=torch.int32, device=device)
        self.rows = 0
        self.blocks = 0

    def append(self, k_rows: torch.Tensor, v_rows: torch.Tensor) -> None:
        n = k_rows.shape[0]
        if self.rows + n > self.capacity:
            raise SpecsvError(abi.EINVAL, "LayerCache: capacity exceeded")
        self.k[self.rows:self.rows + n].copy_(k_rows)
        self.v[self.rows:self.rows + n].copy_(v_rows)
        self.rows += n

    def c(self) -> abi.LayerKvC:
        return abi.LayerKvC(self.k.data_ptr(), self.v.data_ptr(), self.rows, self.ck.data_ptr(),
                            self.ck16.data_ptr(), self.cv.data_ptr(), self.blocks, self.capacity,
                            self.ckd.data_ptr(), self.ckexp.data_ptr())

    def extend_compressed(self, pos_embed: torch.Tensor | None = None, stream=None) -> None:
        """extend_compressed_layer: pool the blocks the new rows complete."""
        want = self.cfg.compressed_block_count(self.rows)
        if want <= self.blocks:
            return
        cfg, kv = self.cfg.c(), self.c()
        check(lib().specsv_compress_append(C.byref(cfg), C.byref(kv), self.blocks, want,
                                           _ptr(pos_embed), _stream(stream)))
        self.blocks = want


@dataclass
class IndexSets:
    """Selected blocks of one (layer, request): [nq][n] int32 ascending, -1
    padded; counts (-1 = no set); forced bitmasks."""
    idx: torch.Tensor
    count: torch.Tensor
    forced: torch.Tensor

    @classmethod
    def empty(cls, nq: int, n: int, device="cuda"):
        return cls(torch.full((nq, n), -1, dtype=torch.int32, device=device),
                   torch.full((nq,), -1, dtype=torch.int32, device=device),
                   torch.zeros((nq,), dtype=torch.int32, device=device))


@dataclass
class DraftBatch:
    """Root + gamma draft queries of one verify call (FlatBatch, draft_tree.hpp:41-48)."""
    pos: np.ndarray              # host int64 [nq]
    tree_mask: np.ndarray        # host uint64 [max(gamma,1)][words]
    q: torch.Tensor              # device fp32 [nq][Hq][dh]
    gates: torch.Tensor          # device fp32 [nq][Hq][3]
    tree_k: torch.Tensor | None  # device bf16 [gamma][Hkv][dh]
    tree_v: torch.Tensor | None
    _keep: list = field(default_factory=list)

    @property
    def n_queries(self) -> int:
        return int(self.q.shape[0])


class Workspace:
    def __init__(self, cfg: NsaConfig, n_queries: int, max_rows: int, device="cuda", batch: int = 1):
        """batch > 1: room for that many REFRESH requests of nsa_verify_batched
        to share one routing launch (specsv_verify_workspace_size_batched)."""
        c = cfg.c()
        if batch > 1:
            self.nbytes = int(lib().specsv_verify_workspace_size_batched(C.byref(c), n_queries,
                                                                          max_rows, batch))
        else:
            self.nbytes = int(lib().specsv_verify_workspace_size(C.byref(c), n_queries, max_rows))
        # zero-filled once: the library keeps its barrier words consistent afterwards
        self.buf = torch.zeros(max(self.nbytes, 256), dtype=torch.uint8, device=device)
        self._fb = int(lib().specsv_debug_route3_counter_offset(C.byref(c), n_queries, max_rows))

    def route_fallbacks(self) -> int:
        """Cumulative exact fp64 re-scorings of the routing kernel on this
        workspace (queries whose certified Top-n boundary fell inside the score
        error bound).  Diagnostics; synchronises."""
        return int(self.buf[4 * self._fb:4 * self._fb + 4].view(torch.int32).item())


def _args(batch: DraftBatch, sets: IndexSets, out: torch.Tensor, group_size: int, mode: int,
          role: int, kv_heads: tuple[int, int] | None = None) -> abi.VerifyArgsC:
    pos = np.ascontiguousarray(batch.pos, np.int64)
    mask = np.ascontiguousarray(batch.tree_mask, np.uint64)
    batch._keep[:] = [pos, mask]
    a = abi.VerifyArgsC()
    a.n_queries = batch.n_queries
    a.group_size = group_size
    a.mode = mode
    a.role = role
    a.pos = pos.ctypes.data_as(C.POINTER(C.c_int64))
    a.tree_mask = mask.ctypes.data_as(C.POINTER(C.c_uint64))
    a.mask_words = mask.shape[1] if mask.ndim == 2 else 1
    a.q = batch.q.data_ptr()
    a.gates = batch.gates.data_ptr()
    a.tree_k = batch.tree_k.data_ptr() if batch.tree_k is not None else None
    a.tree_v = batch.tree_v.data_ptr() if batch.tree_v is not None else None
    a.idx = sets.idx.data_ptr()
    a.idx_count = sets.count.data_ptr()
    a.idx_forced = sets.forced.data_ptr()
    a.out = out.data_ptr()
    if kv_heads is not None:  # KV-head group shard: attend heads [begin, begin + count)
        a.kv_head_begin, a.kv_head_count = int(kv_heads[0]), int(kv_heads[1])
    return a


def _call(fn, cfg, cache, batch, sets, out, ws, group_size, mode, role, stream, kv_heads=None):
    c, kv = cfg.c(), cache.c()
    a = _args(batch, sets, out, group_size, mode, role, kv_heads)
    check(fn(C.byref(c), C.byref(kv), C.byref(a), C.c_void_p(ws.buf.data_ptr()), ws.nbytes,
             _stream(stream)))


def nsa_verify(cfg, cache, batch, sets, out, ws, group_size=4, mode=MODE_EXACT,
               role=ROLE_REFRESH, stream=None, kv_heads=None):
    """One layer of the verify pass (engine.cpp:175-278). REFRESH writes `sets`;
    REUSE reads the source layer's `sets`.  kv_heads=(begin, count): KV-head
    group shard -- routing still scores every head, attention (and `out`) covers
    only that group's heads."""
    _call(lib().specsv_nsa_verify, cfg, cache, batch, sets, out, ws, group_size, mode, role, stream,
          kv_heads)


def nsa_verify_batched(cfg, caches, batches, sets, outs, ws, group_size=4, mode=MODE_EXACT,
                       roles=None, stream=None, kv_heads=None):
    """`len(caches)` independent requests, one layer each, in one call
    (specsv_nsa_verify_batched).  The whole batch is validated before the
    first launch; `ws` must be sized for the largest request."""
    n = len(caches)
    if not (len(batches) == len(sets) == len(outs) == n):
        raise ValueError("caches, batches, sets and outs must have the same length")
    roles = [ROLE_REFRESH] * n if roles is None else list(roles)
    kvs = (abi.LayerKvC * max(n, 1))(*[c.c() for c in caches])
    # kv_heads: None (all heads), one (begin, count) for every request, or a
    # per-request list of (begin, count) / None
    if kv_heads is None:
        heads = [None] * n
    elif len(kv_heads) == 2 and all(isinstance(v, int) for v in kv_heads):
        heads = [tuple(kv_heads)] * n
    else:
        heads = list(kv_heads)
        if len(heads) != n:
            raise ValueError("kv_heads: one entry per request")
    args = (abi.VerifyArgsC * max(n, 1))(*[_args(b, s, o, group_size, mode, r, hh)
                                           for b, s, o, r, hh in zip(batches, sets, outs, roles, heads)])
    c = cfg.c()
    check(lib().specsv_nsa_verify_batched(C.byref(c), kvs, args, n,
                                          C.c_void_p(ws.buf.data_ptr()), ws.nbytes,
                                          _stream(stream)))


class PreparedVerify:
    """nsa_verify / nsa_verify_batched for a fixed set of buffers with the
    ctypes arguments built once: run() refreshes only what changes from step
    to step (committed rows and blocks, positions, tree mask) and calls the
    C-ABI -- the low-overhead form an engine issues every step (same entry
    points, same semantics as nsa_verify)."""

    def __init__(self, cfg, caches, batches, sets, outs, ws, group_size=4, mode=MODE_EXACT,
                 role=ROLE_REFRESH, kv_heads=None):
        one = isinstance(caches, LayerCache)
        self.caches = [caches] if one else list(caches)
        self.batches = [batches] if one else list(batches)
        sets = [sets] if one else list(sets)
        outs = [outs] if one else list(outs)
        heads = [kv_heads] if one or kv_heads is None or isinstance(kv_heads[0], int) \
            else list(kv_heads)
        if len(heads) == 1:
            heads = heads * len(self.caches)
        n = len(self.caches)
        self.cfgc = cfg.c()
        self.kvs = (abi.LayerKvC * n)(*[c.c() for c in self.caches])
        self.args = (abi.VerifyArgsC * n)(*[_args(b, s, o, group_size, mode, role, h)
                                           for b, s, o, h in zip(self.batches, sets, outs, heads)])
        self._keep = [b._keep[:] for b in self.batches]
        self.ws = C.c_void_p(ws.buf.data_ptr())
        self.wsn = ws.nbytes
        self.n = n
        self.fn = lib().specsv_nsa_verify if n == 1 else lib().specsv_nsa_verify_batched

    def run(self, stream=None):
        for i in range(self.n):
            c, b, kv, a = self.caches[i], self.batches[i], self.kvs[i], self.args[i]
            kv.rows = c.rows
            kv.blocks = c.blocks
            if self._keep[i][0] is not b.pos:  # positions / mask replaced since the last step
                pos = np.ascontiguousarray(b.pos, np.int64)
                mask = np.ascontiguousarray(b.tree_mask, np.uint64)
                a.pos = pos.ctypes.data_as(C.POINTER(C.c_int64))
                a.tree_mask = mask.ctypes.data_as(C.POINTER(C.c_uint64))
                a.mask_words = mask.shape[1] if mask.ndim == 2 else 1
                b.pos = pos
                self._keep[i] = [pos, mask]
        st = _stream(stream)
        if self.n == 1:
            check(self.fn(C.byref(self.cfgc), C.byref(self.kvs[0]), C.byref(self.args[0]), self.ws,
                          self.wsn, st))
        else:
            check(self.fn(C.byref(self.cfgc), self.kvs, self.args, self.n, self.ws, self.wsn, st))


def route(cfg, cache, batch, sets, out, ws, group_size=4, mode=MODE_EXACT, stream=None):
    _call(lib().specsv_nsa_route, cfg, cache, batch, sets, out, ws, group_size, mode,
          ROLE_REFRESH, stream)


def attend_fused(cfg, cache, batch, sets, out, ws, group_size=4, mode=MODE_EXACT,
                 role=ROLE_REUSE, stream=None, kv_heads=None):
    _call(lib().specsv_nsa_attend_fused, cfg, cache, batch, sets, out, ws, group_size, mode,
          role, stream, kv_heads)


def selection_scores(cfg, cache, batch, query: int, ws, stream=None) -> torch.Tensor:
    """fp64 selection scores of one query (nsa_attention.cpp:38-80), on device."""
    avail = -(-cfg.routing_visible_len(int(batch.pos[query])) // cfg.l_sel)
    scores = torch.zeros(max(avail, 1), dtype=torch.float64, device=batch.q.device)
    sets = IndexSets.empty(batch.n_queries, cfg.n, batch.q.device)
    out = torch.empty(1, device=batch.q.device)
    c, kv = cfg.c(), cache.c()
    a = _args(batch, sets, out, 1, MODE_EXACT, ROLE_REFRESH)
    check(lib().specsv_nsa_scores(C.byref(c), C.byref(kv), C.byref(a), query,
                                  C.c_void_p(scores.data_ptr()), C.c_void_p(ws.buf.data_ptr()),
                                  ws.nbytes, _stream(stream)))
    return scores[:avail]


def select_blocks(cfg, scores: torch.Tensor, visible_len: int, stream=None):
    """Top-n with forced blocks over device fp64 scores (nsa_attention.cpp:94-136)."""
    dev = scores.device
    idx = torch.full((cfg.n,), -1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    forced = torch.zeros(1, dtype=torch.int32, device=dev)
    c = cfg.c()
    check(lib().specsv_select_blocks(C.byref(c), C.c_void_p(scores.data_ptr()), visible_len,
                                     C.c_void_p(idx.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                     C.c_void_p(forced.data_ptr()), _stream(stream)))
    n = int(cnt.item())
    f = int(forced.item()) & 0xFFFFFFFF
    return idx[:n].tolist(), [bool((f >> i) & 1) for i in range(n)]


def resolve_layer_roles(reuse_set, n_layers: int):
    s = np.ascontiguousarray(list(reuse_set) or [0], np.int64)
    roles = np.zeros(n_layers, np.int32)
    source = np.zeros(n_layers, np.int64)
    check(lib().specsv_resolve_layer_roles(s.ctypes.data_as(C.POINTER(C.c_int64)),
                                           len(list(reuse_set)), n_layers,
                                           roles.ctypes.data_as(C.POINTER(C.c_int32)),
                                           source.ctypes.data_as(C.POINTER(C.c_int64))))
    return roles, source


def clamp_inherited_indices(cfg: NsaConfig, src, forced_bits: int, causal_bound: int):
    s = np.ascontiguousarray(list(src) or [0], np.int32)
    out = np.zeros(max(1, len(list(src))), np.int32)
    of = C.c_uint32(0)
    cnt = C.c_int32(0)
    c = cfg.c()
    check(lib().specsv_clamp_inherited(C.byref(c), s.ctypes.data_as(C.POINTER(C.c_int32)),
                                       forced_bits, len(list(src)), causal_bound,
                                       out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(of),
                                       C.byref(cnt)))
    n = cnt.value
    return out[:n].tolist(), [bool((of.value >> i) & 1) for i in range(n)]


def load_stats(cfg, rows, pos, tree_mask, idx, counts, group_size, mode, role) -> dict:
    pos = np.ascontiguousarray(pos, np.int64)
    mask = np.ascontiguousarray(tree_mask, np.uint64)
    idx = np.ascontiguousarray(idx, np.int32)
    counts = np.ascontiguousarray(counts, np.int32)
    st = abi.LoadStatsC()
    c = cfg.c()
    check(lib().specsv_load_stats(C.byref(c), rows, len(pos),
                                  pos.ctypes.data_as(C.POINTER(C.c_int64)),
                                  mask.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  mask.shape[1] if mask.ndim == 2 else 1, group_size, mode, role,
                                  idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                  counts.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(st)))
    return st.as_dict()


def algorithmic_bytes(cfg, rows, pos, role, idx, counts, mode, group_size) -> int:
    pos = np.ascontiguousarray(pos, np.int64)
    idx = np.ascontiguousarray(idx, np.int32)
    counts = np.ascontiguousarray(counts, np.int32)
    out = C.c_int64(0)
    c = cfg.c()
    check(lib().specsv_algorithmic_bytes(C.byref(c), rows, len(pos),
                                         pos.ctypes.data_as(C.POINTER(C.c_int64)), role,
                                         idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                         counts.ctypes.data_as(C.POINTER(C.c_int32)), mode,
                                         group_size, C.byref(out)))
    return int(out.value)
