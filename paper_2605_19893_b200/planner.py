"""Python face of the host planner policy (include/specsv_b200/planner.h),
mirroring the reference's plan:: and cost:: interfaces.

Reference names (paths relative to /root/reference/proj):
  StrategyTuple, satisfies, validate_strategy, parse_strategy
                                   include/specsv/plan/strategy.hpp:14-45
  bucket_of, ProfileTable, profile_offline, preselect
                                   include/specsv/plan/profile.hpp:15-76
  GuardConstants, RefinerState, refine_step
                                   include/specsv/plan/refiner.hpp:12-62
  CostCoeffs, StepAccounting, account_step, estimate_latency, index_share,
  fit_cost_coeffs                  include/specsv/cost/cost_model.hpp:14-57

All logic runs in the C++ library; this module only marshals arguments.
Errors raise SpecsvError under the conditions where the reference throws
std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

from . import abi
from .abi import SpecsvError, check

NUM_BUCKETS, BUCKET_WIDTH, NUM_CLASSES, CANDIDATES_PER_ENTRY = 4, 4096, 4, 12
MAX_REUSE, MAX_RANKS = 64, 64
MAX_TRANSITIONS, EARLY_WINDOW = 2, 32
STRICT, REUSE_ONLY, APPROX_ONLY, APPROX_REUSE = range(4)
BFS, DFS = 0, 1
EXACT, APPROX = abi.MODE_EXACT, abi.MODE_APPROX

EXPORTED = (
    "specsv_plan_bucket_of", "specsv_plan_satisfies", "specsv_plan_validate_strategy",
    "specsv_plan_parse_strategy", "specsv_plan_strategy_to_string", "specsv_plan_profile_create",
    "specsv_plan_profile_destroy", "specsv_plan_profile_offline", "specsv_plan_profile_put",
    "specsv_plan_profile_entry", "specsv_plan_profile_stored", "specsv_plan_profile_accesses",
    "specsv_plan_preselect", "specsv_plan_refiner_init", "specsv_plan_refine_step",
    "specsv_plan_observed_throughput", "specsv_cost_default_coeffs", "specsv_cost_validate",
    "specsv_cost_account_step", "specsv_cost_estimate_latency", "specsv_cost_index_share",
    "specsv_cost_fit",
)


class StrategyC(C.Structure):
    _fields_ = [("depth", C.c_int64), ("width", C.c_int64), ("traversal", C.c_int32),
                ("mode", C.c_int32), ("group_size", C.c_int64), ("budget", C.c_int64),
                ("n_reuse", C.c_int32), ("reserved", C.c_int32),
                ("reuse_set", C.c_int64 * MAX_REUSE)]


class CandidateC(C.Structure):
    _fields_ = [("strategy", StrategyC), ("exp_accepted", C.c_double),
                ("exp_latency", C.c_double), ("throughput", C.c_double)]


class GuardConstantsC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("rho", C.c_double), ("warmup", C.c_int64),
                ("hysteresis", C.c_int64)]


class RefinerStateC(C.Structure):
    _fields_ = [("consts", GuardConstantsC), ("ema", C.c_double), ("ema_primed", C.c_int32),
                ("settled", C.c_int32), ("steps_seen", C.c_int64), ("below_count", C.c_int64),
                ("transitions", C.c_int64), ("active_rank", C.c_int64),
                ("n_explored", C.c_int32), ("reserved", C.c_int32),
                ("explored_rank", C.c_int64 * MAX_RANKS),
                ("explored_sum_accepted", C.c_double * MAX_RANKS),
                ("explored_sum_latency", C.c_double * MAX_RANKS),
                ("explored_steps", C.c_int64 * MAX_RANKS)]


class DecisionC(C.Structure):
    _fields_ = [("switched", C.c_int32), ("settled_now", C.c_int32), ("active_rank", C.c_int64)]


class CostCoeffsC(C.Structure):
    _fields_ = [("c_block", C.c_double), ("c_index", C.c_double), ("c_launch", C.c_double),
                ("c_window", C.c_double), ("c_base", C.c_double)]


class StepAccountingC(C.Structure):
    _fields_ = [("unique_loads", C.c_int64), ("constructions", C.c_int64),
                ("launches", C.c_int64), ("window_tokens", C.c_int64), ("layers", C.c_int64)]


class FitSampleC(C.Structure):
    _fields_ = [("acc", StepAccountingC), ("measured", C.c_double)]


EVAL_FN = C.CFUNCTYPE(C.c_int32, C.POINTER(StrategyC), C.c_int32, C.c_int32,
                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32, C.c_void_p)

_ready = False


def _lib() -> C.CDLL:
    global _ready
    L = abi.lib()
    if _ready:
        return L
    i32, i64, dbl, vp, sz = C.c_int32, C.c_int64, C.c_double, C.c_void_p, C.c_size_t
    sp, cp = C.POINTER(StrategyC), C.POINTER(CandidateC)
    rsp, accp, coefp = C.POINTER(RefinerStateC), C.POINTER(StepAccountingC), C.POINTER(CostCoeffsC)
    sig = {
        "specsv_plan_bucket_of": ([i64], i32),
        "specsv_plan_satisfies": ([sp, i32], i32),
        "specsv_plan_validate_strategy": ([sp, i32], C.c_int),
        "specsv_plan_parse_strategy": ([C.c_char_p, sp], C.c_int),
        "specsv_plan_strategy_to_string": ([sp, C.c_char_p, sz], C.c_int),
        "specsv_plan_profile_create": ([], vp),
        "specsv_plan_profile_destroy": ([vp], None),
        "specsv_plan_profile_offline": ([EVAL_FN, vp, sp, i32, i32, vp], C.c_int),
        "specsv_plan_profile_put": ([vp, i32, i32, cp, i32], C.c_int),
        "specsv_plan_profile_entry": ([vp, i32, i32, cp, i32, C.POINTER(i32)], C.c_int),
        "specsv_plan_profile_stored": ([vp], i64),
        "specsv_plan_profile_accesses": ([vp, i64], i64),
        "specsv_plan_preselect": ([vp, i32, i32, cp], C.c_int),
        "specsv_plan_refiner_init": ([rsp], None),
        "specsv_plan_refine_step": ([rsp, dbl, dbl, C.POINTER(dbl), i32, C.POINTER(DecisionC)],
                                    C.c_int),
        "specsv_plan_observed_throughput": ([rsp, i64], dbl),
        "specsv_cost_default_coeffs": ([coefp], None),
        "specsv_cost_validate": ([coefp], C.c_int),
        "specsv_cost_account_step": ([C.POINTER(abi.LoadStatsC), i64, C.POINTER(i64), i64, accp],
                                     C.c_int),
        "specsv_cost_estimate_latency": ([accp, coefp], dbl),
        "specsv_cost_index_share": ([accp, coefp], dbl),
        "specsv_cost_fit": ([C.POINTER(FitSampleC), i64, coefp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _ready = True
    return L


# ---------------------------------------------------------------- strategy
@dataclass
class StrategyTuple:
    depth: int = 4
    width: int = 2
    traversal: int = BFS
    group_size: int = 2
    mode: int = EXACT
    reuse_set: List[int] = field(default_factory=list)
    budget: Optional[int] = None

    def c(self) -> StrategyC:
        if len(self.reuse_set) > MAX_REUSE:
            raise SpecsvError(abi.EUNSUPPORTED, "reuse set longer than this build carries")
        s = StrategyC(self.depth, self.width, self.traversal, self.mode, self.group_size,
                      -1 if self.budget is None else self.budget, len(self.reuse_set), 0)
        for i, j in enumerate(self.reuse_set):
            s.reuse_set[i] = j
        return s

    @staticmethod
    def from_c(s: StrategyC) -> "StrategyTuple":
        return StrategyTuple(s.depth, s.width, s.traversal, s.group_size, s.mode,
                             [s.reuse_set[i] for i in range(s.n_reuse)],
                             None if s.budget < 0 else s.budget)

    def to_string(self) -> str:
        buf = C.create_string_buffer(512)
        check(_lib().specsv_plan_strategy_to_string(C.byref(self.c()), buf, 512))
        return buf.value.decode()


def bucket_of(context_len: int) -> int:
    b = _lib().specsv_plan_bucket_of(context_len)
    if b < 0:
        raise SpecsvError(abi.EINVAL, abi.lib().specsv_last_error().decode())
    return b


def satisfies(s: StrategyTuple, cls: int) -> bool:
    return bool(_lib().specsv_plan_satisfies(C.byref(s.c()), cls))


def validate_strategy(s: StrategyTuple, cls: int) -> None:
    check(_lib().specsv_plan_validate_strategy(C.byref(s.c()), cls))


def parse_strategy(text: str) -> StrategyTuple:
    out = StrategyC()
    check(_lib().specsv_plan_parse_strategy(text.encode(), C.byref(out)))
    return StrategyTuple.from_c(out)


# ---------------------------------------------------------------- profile
@dataclass
class ProfiledCandidate:
    strategy: StrategyTuple
    exp_accepted: float
    exp_latency: float
    throughput: float


@dataclass
class EvalTrace:
    step_accepted: List[float]
    step_latency: List[float]


class ProfileTable:
    """Owns the library's table; entries are read through `at` (one counted
    access, ProfileTable::at) or `grid(b, c)` (uncounted, for inspection)."""

    def __init__(self):
        self._h = C.c_void_p(_lib().specsv_plan_profile_create())

    def __del__(self):
        if getattr(self, "_h", None):
            _lib().specsv_plan_profile_destroy(self._h)
            self._h = None

    def _entry(self, bucket: int, cls: int) -> List[ProfiledCandidate]:
        buf = (CandidateC * CANDIDATES_PER_ENTRY)()
        n = C.c_int32()
        check(_lib().specsv_plan_profile_entry(self._h, bucket, cls, buf, CANDIDATES_PER_ENTRY,
                                               C.byref(n)))
        return [ProfiledCandidate(StrategyTuple.from_c(buf[i].strategy), buf[i].exp_accepted,
                                  buf[i].exp_latency, buf[i].throughput) for i in range(n.value)]

    def at(self, bucket: int, cls: int) -> List[ProfiledCandidate]:
        return self._entry(bucket, cls)

    def grid(self, bucket: int, cls: int) -> List[ProfiledCandidate]:
        before = self.entry_accesses
        out = self._entry(bucket, cls)
        self.entry_accesses = before
        return out

    def put(self, bucket: int, cls: int, candidates: Sequence[ProfiledCandidate]) -> None:
        buf = (CandidateC * max(1, len(candidates)))()
        for i, c in enumerate(candidates):
            buf[i] = CandidateC(c.strategy.c(), c.exp_accepted, c.exp_latency, c.throughput)
        check(_lib().specsv_plan_profile_put(self._h, bucket, cls, buf, len(candidates)))

    def stored_strategies(self) -> int:
        return _lib().specsv_plan_profile_stored(self._h)

    @property
    def entry_accesses(self) -> int:
        return _lib().specsv_plan_profile_accesses(self._h, -1)

    @entry_accesses.setter
    def entry_accesses(self, value: int) -> None:
        _lib().specsv_plan_profile_accesses(self._h, value)


def profile_offline(evaluate: Callable[[StrategyTuple, int, int], EvalTrace],
                    candidates: Sequence[StrategyTuple], max_steps: int = 256) -> ProfileTable:
    """profile_offline (profile.cpp:60-96) with a Python evaluator."""
    err: List[BaseException] = []

    def cb(sp, bucket, cls, acc, lat, cap, _user):
        try:
            tr = evaluate(StrategyTuple.from_c(sp.contents), bucket, cls)
            if len(tr.step_accepted) != len(tr.step_latency):
                return 0  # ragged: the library rejects an empty trace
            n = min(cap, len(tr.step_accepted))
            for i in range(n):
                acc[i] = tr.step_accepted[i]
                lat[i] = tr.step_latency[i]
            return n
        except BaseException as e:  # noqa: BLE001 -- re-raised after the call
            err.append(e)
            return -1

    fn = EVAL_FN(cb)
    arr = (StrategyC * max(1, len(candidates)))(*[s.c() for s in candidates])
    table = ProfileTable()
    status = _lib().specsv_plan_profile_offline(fn, None, arr, len(candidates), max_steps,
                                                table._h)
    if err:
        raise err[0]
    check(status)
    return table


def preselect(table: ProfileTable, bucket: int, cls: int) -> ProfiledCandidate:
    out = CandidateC()
    check(_lib().specsv_plan_preselect(table._h, bucket, cls, C.byref(out)))
    return ProfiledCandidate(StrategyTuple.from_c(out.strategy), out.exp_accepted,
                             out.exp_latency, out.throughput)


# ---------------------------------------------------------------- refiner
@dataclass
class GuardConstants:
    alpha: float = 0.40
    rho: float = 0.85
    warmup: int = 8
    hysteresis: int = 5


@dataclass
class RefineDecision:
    switched: bool
    settled_now: bool
    active_rank: int


class RefinerState:
    """Per-request guard state (refiner.hpp:26-44), held by the library."""

    def __init__(self, consts: Optional[GuardConstants] = None):
        self._s = RefinerStateC()
        _lib().specsv_plan_refiner_init(C.byref(self._s))
        if consts is not None:
            self.consts = consts

    @property
    def consts(self) -> GuardConstants:
        c = self._s.consts
        return GuardConstants(c.alpha, c.rho, c.warmup, c.hysteresis)

    @consts.setter
    def consts(self, g: GuardConstants) -> None:
        self._s.consts = GuardConstantsC(g.alpha, g.rho, g.warmup, g.hysteresis)

    def __getattr__(self, name):
        if name in ("ema", "steps_seen", "below_count", "transitions", "active_rank"):
            return getattr(self._s, name)
        if name in ("ema_primed", "settled"):
            return bool(getattr(self._s, name))
        raise AttributeError(name)

    def observed_throughput(self, rank: int) -> float:
        return _lib().specsv_plan_observed_throughput(C.byref(self._s), rank)


def refine_step(state: RefinerState, accepted: float, latency: float,
                entry: Sequence[ProfiledCandidate]) -> RefineDecision:
    exp = (C.c_double * max(1, len(entry)))(*[c.exp_accepted for c in entry])
    d = DecisionC()
    check(_lib().specsv_plan_refine_step(C.byref(state._s), accepted, latency, exp, len(entry),
                                         C.byref(d)))
    return RefineDecision(bool(d.switched), bool(d.settled_now), d.active_rank)


# ---------------------------------------------------------------- cost model
@dataclass
class CostCoeffs:
    c_block: float = 1.0
    c_index: float = 4.0
    c_launch: float = 0.5
    c_window: float = 0.02
    c_base: float = 10.0

    def c(self) -> CostCoeffsC:
        return CostCoeffsC(self.c_block, self.c_index, self.c_launch, self.c_window, self.c_base)

    def validate(self) -> None:
        check(_lib().specsv_cost_validate(C.byref(self.c())))


@dataclass
class StepAccounting:
    unique_loads: int = 0
    constructions: int = 0
    launches: int = 0
    window_tokens: int = 0
    layers: int = 0

    def c(self) -> StepAccountingC:
        return StepAccountingC(self.unique_loads, self.constructions, self.launches,
                               self.window_tokens, self.layers)


def account_step(per_layer: Sequence[dict], reuse_set: Sequence[int], n_layers: int) -> StepAccounting:
    """account_step over per-layer LoadStats dicts (verify.load_stats output
    or hand-built {unique_block_loads, index_constructions, window_token_loads})."""
    arr = (abi.LoadStatsC * max(1, len(per_layer)))()
    for i, s in enumerate(per_layer):
        arr[i].unique_block_loads = s.get("unique_block_loads", 0)
        arr[i].total_requested_loads = s.get("total_requested_loads", 0)
        arr[i].index_constructions = s.get("index_constructions", 0)
        arr[i].window_token_loads = s.get("window_token_loads", 0)
    if len(per_layer) != n_layers:
        raise SpecsvError(abi.EINVAL, "account_step: stats must cover every layer")
    S = (C.c_int64 * max(1, len(reuse_set)))(*reuse_set)
    out = StepAccountingC()
    check(_lib().specsv_cost_account_step(arr, n_layers, S, len(reuse_set), C.byref(out)))
    return StepAccounting(out.unique_loads, out.constructions, out.launches, out.window_tokens,
                          out.layers)


def estimate_latency(acc: StepAccounting, coeffs: CostCoeffs) -> float:
    return _lib().specsv_cost_estimate_latency(C.byref(acc.c()), C.byref(coeffs.c()))


def index_share(acc: StepAccounting, coeffs: CostCoeffs) -> float:
    return _lib().specsv_cost_index_share(C.byref(acc.c()), C.byref(coeffs.c()))


def fit_cost_coeffs(samples: Sequence[tuple]) -> CostCoeffs:
    """samples: (StepAccounting, measured latency) pairs."""
    arr = (FitSampleC * max(1, len(samples)))()
    for i, (acc, t) in enumerate(samples):
        arr[i] = FitSampleC(acc.c(), t)
    out = CostCoeffsC()
    check(_lib().specsv_cost_fit(arr, len(samples), C.byref(out)))
    return CostCoeffs(out.c_block, out.c_index, out.c_launch, out.c_window, out.c_base)
