"""Python face of the draft-tree utilities and the accepted-row commit
(include/specsv_b200/draft_tree.h), mirroring the reference's tree:: interface
and the commit loop of Engine::step.

Reference names (paths relative to /root/reference/proj):
  DraftNode, DraftTree, Traversal, FlatBatch, TokenScore, ProposeFn,
  expand_draft_tree, flatten_tree, build_tree_mask, VerifyResult,
  greedy_verify                     include/specsv/tree/draft_tree.hpp:14-90
                                    src/draft_tree.cpp:45-164
  commit of accepted scratch rows   src/engine.cpp:533-547

All logic runs in the C++ library (the commit on the GPU); this module only
marshals arguments.  FlatBatch.mask is the boundary's packed form (uint64
[gamma][ceil(gamma / 64)], bit j of row i = mask[i][j]); `mask_bool()` gives
the reference's vector<vector<bool>> view.  Errors raise SpecsvError where
the reference throws std::invalid_argument (or asserts).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import abi
from .abi import SpecsvError, check

BFS, DFS = 0, 1
NO_PARENT = -1

EXPORTED = ("specsv_tree_expand", "specsv_tree_flatten", "specsv_tree_mask",
            "specsv_tree_greedy_accept", "specsv_commit_rows", "specsv_commit_rows_compress")


class DraftTreeC(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("parent", C.POINTER(C.c_int64)),
                ("token", C.POINTER(C.c_int32)), ("depth", C.POINTER(C.c_int32)),
                ("score", C.POINTER(C.c_double))]


PROPOSE_FN = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                         C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_double))

_ready = False


def _lib() -> C.CDLL:
    global _ready
    L = abi.lib()
    if _ready:
        return L
    i32, i64, vp = C.c_int32, C.c_int64, C.c_void_p
    i64p, i32p, dp, u64p = (C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                            C.POINTER(C.c_uint64))
    tp = C.POINTER(DraftTreeC)
    sig = {
        "specsv_tree_expand": ([i32, PROPOSE_FN, vp, i64, i64, i64, i64, i64p, i32p, i32p, dp, dp,
                                i64p], C.c_int),
        "specsv_tree_flatten": ([tp, i32, i64, i64p, i64p, u64p, i32], C.c_int),
        "specsv_tree_mask": ([tp, i64p, i64, u64p, i32], C.c_int),
        "specsv_tree_greedy_accept": ([tp, i32p, i64p, i32p, i64p, i32p], C.c_int),
        "specsv_commit_rows": ([C.POINTER(abi.NsaConfigC), C.POINTER(abi.LayerKvC),
                                C.POINTER(vp), C.POINTER(vp), i32, i32p, i32, vp], C.c_int),
        "specsv_commit_rows_compress": ([C.POINTER(abi.NsaConfigC), C.POINTER(abi.LayerKvC),
                                         C.POINTER(vp), C.POINTER(vp), i32, i32p, i32, C.POINTER(vp),
                                         vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _ready = True
    return L


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


@dataclass
class TokenScore:
    token: int
    score: float


@dataclass
class DraftTree:
    """DraftTree (draft_tree.hpp:28-34) as flat node arrays; node 0 is the root."""
    parent: np.ndarray                      # int64 [n]
    token: np.ndarray                       # int32 [n]
    depth: np.ndarray                       # int32 [n]
    score: np.ndarray                       # float64 [n]
    cum_score: Optional[np.ndarray] = None  # float64 [n]

    @classmethod
    def from_nodes(cls, nodes: Sequence[tuple]) -> "DraftTree":
        """nodes = [(parent, token, score), ...] with node 0 the root (parent -1);
        depth and cum_score follow from the parents (tree_from_json,
        draft_tree.cpp:185-212)."""
        n = len(nodes)
        parent = np.array([p for p, _, _ in nodes], np.int64)
        token = np.array([t for _, t, _ in nodes], np.int32)
        score = np.array([s for _, _, s in nodes], np.float64)
        depth = np.zeros(n, np.int32)
        cum = np.zeros(n, np.float64)
        for i in range(1, n):
            p = int(parent[i])
            if not 0 <= p < i:
                raise SpecsvError(abi.EINVAL, f"node {i}: parent must precede it")
            depth[i] = depth[p] + 1
            cum[i] = cum[p] + score[i]
        return cls(parent, token, depth, score, cum)

    @property
    def n_nodes(self) -> int:
        return int(self.parent.shape[0])

    @property
    def gamma(self) -> int:
        return self.n_nodes - 1

    def children(self, node: int) -> List[int]:
        return [i for i in range(1, self.n_nodes) if int(self.parent[i]) == node]

    def is_ancestor_or_self(self, anc: int, node: int) -> bool:
        cur = node
        while cur != NO_PARENT:
            if cur == anc:
                return True
            cur = int(self.parent[cur])
        return False

    def c(self) -> DraftTreeC:
        self.parent = np.ascontiguousarray(self.parent, np.int64)
        self.token = np.ascontiguousarray(self.token, np.int32)
        self.depth = np.ascontiguousarray(self.depth, np.int32)
        self.score = np.ascontiguousarray(self.score, np.float64)
        return DraftTreeC(self.n_nodes, _p(self.parent, C.c_int64), _p(self.token, C.c_int32),
                          _p(self.depth, C.c_int32), _p(self.score, C.c_double))


@dataclass
class FlatBatch:
    """FlatBatch (draft_tree.hpp:41-48) with the mask in the boundary's packed form."""
    traversal: int
    order: np.ndarray      # int64 [gamma] node ids
    positions: np.ndarray  # int64 [gamma] committed_len - 1 + depth
    mask: np.ndarray       # uint64 [gamma][words]
    gamma: int

    def mask_bool(self) -> np.ndarray:
        return unpack_mask(self.mask, self.gamma)


@dataclass
class VerifyResult:
    """VerifyResult (draft_tree.hpp:79-85)."""
    accepted_nodes: List[int] = field(default_factory=list)
    accepted_tokens: List[int] = field(default_factory=list)
    bonus_token: int = 0

    @property
    def accepted_count(self) -> int:
        return len(self.accepted_tokens) + 1


def mask_words(gamma: int) -> int:
    return max(1, (gamma + 63) // 64)


def unpack_mask(mask: np.ndarray, gamma: int) -> np.ndarray:
    out = np.zeros((gamma, gamma), bool)
    for i in range(gamma):
        for j in range(gamma):
            out[i, j] = bool((int(mask[i, j // 64]) >> (j % 64)) & 1)
    return out


def expand_draft_tree(root_token: int, propose: Callable[[int, int, int, float, int],
                                                         Sequence[TokenScore]],
                      D: int, k: int, budget: Optional[int] = None) -> DraftTree:
    """expand_draft_tree (draft_tree.cpp:45-82).  propose(node_id, token, depth,
    cum_score, k) returns the draft model's top-k TokenScores (distinct tokens,
    descending score)."""
    if D >= 1 and k >= 1:
        full = sum(k ** d for d in range(D + 1))
        cap = full if budget is None else min(full, budget + 1)
    else:
        cap = 1
    parent = np.zeros(cap, np.int64)
    token = np.zeros(cap, np.int32)
    depth = np.zeros(cap, np.int32)
    score = np.zeros(cap, np.float64)
    cum = np.zeros(cap, np.float64)
    err: list = []

    def cb(_ctx, node, tok, dep, cs, kk, tok_out, sc_out):
        try:
            top = list(propose(int(node), int(tok), int(dep), float(cs), int(kk)))
            if len(top) > kk:
                return -1
            for i, ts in enumerate(top):
                tok_out[i] = int(ts.token)
                sc_out[i] = float(ts.score)
            return len(top)
        except Exception as e:  # surfaced after the call
            err.append(e)
            return -1

    fn = PROPOSE_FN(cb)
    n = C.c_int64(0)
    st = _lib().specsv_tree_expand(int(root_token), fn, None, int(D), int(k),
                                   -1 if budget is None else int(budget), cap,
                                   _p(parent, C.c_int64), _p(token, C.c_int32),
                                   _p(depth, C.c_int32), _p(score, C.c_double),
                                   _p(cum, C.c_double), C.byref(n))
    if err:
        raise err[0]
    check(st)
    m = n.value
    return DraftTree(parent[:m].copy(), token[:m].copy(), depth[:m].copy(), score[:m].copy(),
                     cum[:m].copy())


def flatten_tree(tree: DraftTree, traversal: int, committed_len: int) -> FlatBatch:
    """flatten_tree (draft_tree.cpp:84-124) plus build_tree_mask (:126-141)."""
    g = tree.gamma
    words = mask_words(g)
    order = np.zeros(max(g, 1), np.int64)
    pos = np.zeros(max(g, 1), np.int64)
    mask = np.zeros((max(g, 1), words), np.uint64)
    t = tree.c()
    check(_lib().specsv_tree_flatten(C.byref(t), int(traversal), int(committed_len),
                                     _p(order, C.c_int64), _p(pos, C.c_int64),
                                     _p(mask, C.c_uint64), words))
    return FlatBatch(int(traversal), order[:g], pos[:g], mask[:g], g)


def build_tree_mask(tree: DraftTree, order: Sequence[int]) -> np.ndarray:
    """build_tree_mask (draft_tree.cpp:126-141), packed."""
    o = np.ascontiguousarray(np.asarray(order, np.int64))
    g = int(o.shape[0])
    words = mask_words(g)
    mask = np.zeros((max(g, 1), words), np.uint64)
    t = tree.c()
    check(_lib().specsv_tree_mask(C.byref(t), _p(o, C.c_int64), g, _p(mask, C.c_uint64), words))
    return mask[:g]


def greedy_verify(tree: DraftTree, target_argmax: Sequence[int]) -> VerifyResult:
    """greedy_verify (draft_tree.cpp:143-164)."""
    am = np.ascontiguousarray(np.asarray(target_argmax, np.int32))
    if am.shape[0] < tree.n_nodes:
        raise SpecsvError(abi.EINVAL, "greedy_verify: argmax missing for some nodes")
    nodes = np.zeros(max(tree.gamma, 1), np.int64)
    toks = np.zeros(max(tree.gamma, 1), np.int32)
    na, bonus = C.c_int64(0), C.c_int32(0)
    t = tree.c()
    check(_lib().specsv_tree_greedy_accept(C.byref(t), _p(am, C.c_int32), _p(nodes, C.c_int64),
                                           _p(toks, C.c_int32), C.byref(na), C.byref(bonus)))
    return VerifyResult([int(x) for x in nodes[:na.value]], [int(x) for x in toks[:na.value]],
                        int(bonus.value))


def commit_accepted(cfg, caches, tree_ks, tree_vs, slots: Sequence[int], pos_embed=None,
                    stream=None) -> None:
    """Engine::step's commit (engine.cpp:533-547) for every layer at once: the
    accepted draft rows (flat slots, root-to-leaf order) go to committed rows
    [rows, rows + len(slots)) of each LayerCache (one GPU launch), then the
    rows advance and the new compressed blocks are pooled.  pos_embed: one
    device tensor for every layer, or a per-layer sequence."""
    from .verify import _stream  # noqa: PLC0415  (torch-side helpers)
    n = len(caches)
    if not (len(tree_ks) == len(tree_vs) == n):
        raise ValueError("caches, tree_ks and tree_vs must have the same length")
    s = np.ascontiguousarray(np.asarray(slots, np.int32))
    for c in caches:
        if c.rows + len(s) > c.capacity:
            raise SpecsvError(abi.EINVAL, "commit exceeds the cache capacity")
    kvs = (abi.LayerKvC * max(n, 1))(*[c.c() for c in caches])
    tk = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in tree_ks])
    tv = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in tree_vs])
    pes = list(pos_embed) if isinstance(pos_embed, (list, tuple)) else [pos_embed] * n
    pe = (C.c_void_p * max(n, 1))(*[None if x is None else x.data_ptr() for x in pes])
    c = cfg.c()
    # the commit and the compressed blocks it completes, every layer, two launches
    check(_lib().specsv_commit_rows_compress(C.byref(c), kvs, tk, tv, n, _p(s, C.c_int32),
                                             int(s.shape[0]), pe, _stream(stream)))
    for cache in caches:
        cache.rows += int(s.shape[0])
        cache.blocks = cfg.compressed_block_count(cache.rows)


class PreparedCommit:
    """commit_accepted for a fixed set of caches and draft-row buffers with the
    ctypes arguments built once: run() refreshes the committed rows and blocks
    and calls specsv_commit_rows_compress (the form an engine issues every
    step; same entry point and semantics as commit_accepted)."""

    def __init__(self, cfg, caches, tree_ks, tree_vs, slots: Sequence[int], pos_embed=None):
        n = len(caches)
        if not (len(tree_ks) == len(tree_vs) == n):
            raise ValueError("caches, tree_ks and tree_vs must have the same length")
        self.cfg, self.caches, self.n = cfg, list(caches), n
        self.s = np.ascontiguousarray(np.asarray(slots, np.int32))
        self.kvs = (abi.LayerKvC * max(n, 1))(*[c.c() for c in caches])
        self.tk = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in tree_ks])
        self.tv = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in tree_vs])
        pes = list(pos_embed) if isinstance(pos_embed, (list, tuple)) else [pos_embed] * n
        self.pe = (C.c_void_p * max(n, 1))(*[None if x is None else x.data_ptr() for x in pes])
        self.cfgc = cfg.c()
        self.fn = _lib().specsv_commit_rows_compress

    def run(self, stream=None) -> None:
        from .verify import _stream  # noqa: PLC0415
        k = int(self.s.shape[0])
        for i, c in enumerate(self.caches):
            if c.rows + k > c.capacity:
                raise SpecsvError(abi.EINVAL, "commit exceeds the cache capacity")
            self.kvs[i].rows = c.rows
            self.kvs[i].blocks = c.blocks
        check(self.fn(C.byref(self.cfgc), self.kvs, self.tk, self.tv, self.n, _p(self.s, C.c_int32), k,
                      self.pe, _stream(stream)))
        for c in self.caches:
            c.rows += k
            c.blocks = self.cfg.compressed_block_count(c.rows)
