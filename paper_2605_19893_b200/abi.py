"""ctypes binding of the C-ABI (include/specsv_b200/nsa_verify.h).

The library is built in-tree for sm_100a (``python -m paper_2605_19893_b200.build``).
There is no CPU fallback: importing the binding without the built library
raises, and every call returns the library's status code (non-zero raises
``SpecsvError`` with the library's thread-local message).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SPECSV_LIB: diagnostics only (A/B timing of build variants); the default is the in-tree build
LIB_PATH = os.environ.get("SPECSV_LIB") or os.path.join(PKG, "lib", "libspecsv_b200.so")

OK, EINVAL, ESTATE, EUNSUPPORTED, ECUDA, ENOSPACE = range(6)
MODE_EXACT, MODE_APPROX = 0, 1
ROLE_REFRESH, ROLE_REUSE = 0, 1
MAX_PAIRS = 128

EXPORTED = (
    "specsv_abi_version", "specsv_last_error", "specsv_validate_config",
    "specsv_verify_workspace_size", "specsv_verify_workspace_size_batched", "specsv_nsa_verify",
    "specsv_nsa_verify_batched",
    "specsv_nsa_route", "specsv_nsa_attend_fused", "specsv_nsa_scores", "specsv_select_blocks",
    "specsv_compress_append", "specsv_resolve_layer_roles", "specsv_clamp_inherited",
    "specsv_load_stats", "specsv_algorithmic_bytes", "specsv_debug_attend_trace",
    "specsv_debug_route3_counter_offset",
)


class SpecsvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"specsv status {code}: {msg}")
        self.code = code


class NsaConfigC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("l", "d", "l_sel", "n", "w", "n_q_heads", "n_kv_heads", "d_head", "n_layers",
                 "routing_lag")]


class LayerKvC(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("rows", C.c_int64),
                ("ck", C.c_void_p), ("ck16", C.c_void_p), ("cv", C.c_void_p),
                ("blocks", C.c_int64), ("capacity", C.c_int64),
                ("ckd", C.c_void_p), ("ckexp", C.c_void_p)]


class VerifyArgsC(C.Structure):
    _fields_ = [("n_queries", C.c_int32), ("group_size", C.c_int32), ("mode", C.c_int32),
                ("role", C.c_int32), ("pos", C.POINTER(C.c_int64)),
                ("tree_mask", C.POINTER(C.c_uint64)), ("mask_words", C.c_int32),
                ("q", C.c_void_p), ("gates", C.c_void_p), ("tree_k", C.c_void_p),
                ("tree_v", C.c_void_p), ("idx", C.c_void_p), ("idx_count", C.c_void_p),
                ("idx_forced", C.c_void_p), ("out", C.c_void_p),
                ("kv_head_begin", C.c_int32), ("kv_head_count", C.c_int32)]


class LoadStatsC(C.Structure):
    _fields_ = [("unique_block_loads", C.c_int64), ("total_requested_loads", C.c_int64),
                ("dedup_savings", C.c_int64), ("window_token_loads", C.c_int64),
                ("launches", C.c_int64), ("index_constructions", C.c_int64),
                ("n_pairs", C.c_int64), ("pairwise_overlap", C.c_int64 * MAX_PAIRS)]

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


_lib = None


def lib() -> C.CDLL:
    """Loads the sm_100a library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2605_19893_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    cfgp, kvp, argp = C.POINTER(NsaConfigC), C.POINTER(LayerKvC), C.POINTER(VerifyArgsC)
    i32, i64, u32, vp, sz = C.c_int32, C.c_int64, C.c_uint32, C.c_void_p, C.c_size_t
    i64p, i32p, u32p, u64p = (C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
                              C.POINTER(C.c_uint64))
    sig = {
        "specsv_abi_version": ([], i32),
        "specsv_last_error": ([], C.c_char_p),
        "specsv_validate_config": ([cfgp], C.c_int),
        "specsv_verify_workspace_size": ([cfgp, i32, i64], sz),
        "specsv_verify_workspace_size_batched": ([cfgp, i32, i64, i32], sz),
        "specsv_nsa_verify": ([cfgp, kvp, argp, vp, sz, vp], C.c_int),
        "specsv_nsa_verify_batched": ([cfgp, kvp, argp, i32, vp, sz, vp], C.c_int),
        "specsv_nsa_route": ([cfgp, kvp, argp, vp, sz, vp], C.c_int),
        "specsv_nsa_attend_fused": ([cfgp, kvp, argp, vp, sz, vp], C.c_int),
        "specsv_nsa_scores": ([cfgp, kvp, argp, i32, vp, vp, sz, vp], C.c_int),
        "specsv_select_blocks": ([cfgp, vp, i64, vp, vp, vp, vp], C.c_int),
        "specsv_compress_append": ([cfgp, kvp, i64, i64, vp, vp], C.c_int),
        "specsv_resolve_layer_roles": ([i64p, i64, i64, i32p, i64p], C.c_int),
        "specsv_clamp_inherited": ([cfgp, i32p, u32, i32, i64, i32p, u32p, i32p], C.c_int),
        "specsv_load_stats": ([cfgp, i64, i32, i64p, u64p, i32, i32, i32, i32, i32p, i32p,
                               C.POINTER(LoadStatsC)], C.c_int),
        "specsv_algorithmic_bytes": ([cfgp, i64, i32, i64p, i32, i32p, i32p, i32, i32, i64p],
                                     C.c_int),
        "specsv_debug_attend_trace": ([vp], C.c_int),
        "specsv_debug_route3_counter_offset": ([cfgp, i32, i64], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int) -> None:
    if status != OK:
        raise SpecsvError(status, lib().specsv_last_error().decode())
