"""Host planner policy (include/specsv_b200/planner.h) against the reference's
own planner and cost-model tests (tests/test_planner.cpp,
tests/test_cost_model.cpp under /root/reference/proj), re-run through the
C-ABI.  Pure host code: no GPU."""
import os
import re

import pytest

from paper_2605_19893_b200 import abi
from paper_2605_19893_b200 import planner as P

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "specsv_b200",
                      "planner.h")


class Rng:
    """splitmix64 stream (include/specsv/rng.hpp:13-33)."""

    def __init__(self, seed):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def next_unit(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n):
        return 0 if n == 0 else self.next_u64() % n


def default_candidates():  # test_planner.cpp:19-41
    out = []
    shapes = [(1, 1), (2, 2), (4, 2), (6, 2), (4, 4), (6, 4)]
    for mode in (P.EXACT, P.APPROX):
        for reuse in (0, 1):
            i = 0
            for d, k in shapes:
                for t in (P.BFS, P.DFS):
                    out.append(P.StrategyTuple(d, k, t, 2 if i % 2 == 0 else 4, mode,
                                               [1, 3] if reuse else []))
                    i += 1
    return out


def fake_eval(s, bucket, cls, log=None):  # test_planner.cpp:45-62
    rng = Rng(s.depth * 1000 + s.width * 100 + s.group_size * 10 + bucket +
              (0 if s.traversal == P.BFS else 7) + (0 if s.mode == P.EXACT else 13) +
              (0 if not s.reuse_set else 29))
    base_a = 1.0 + 0.4 * min(s.depth, 5)
    base_t = (1.0 + 0.08 * (s.depth * s.width) + 0.25 * bucket - (0.0 if not s.reuse_set else 0.2)
              - (0.1 if s.mode == P.APPROX else 0.0))
    tr = P.EvalTrace([], [])
    for _ in range(6):
        tr.step_accepted.append(base_a + 0.2 * rng.next_unit())
        tr.step_latency.append(base_t + 0.05 * rng.next_unit())
    if log is not None:
        log.append((bucket, cls, s, tr))
    return tr


def entry_with_expectations(exp_a):  # test_planner.cpp:64-78
    return [P.ProfiledCandidate(P.StrategyTuple(depth=i + 1), a, 1.0, a)
            for i, a in enumerate(exp_a)]


def run_trace(st, entry, accepted):  # test_planner.cpp:80-90
    switches = []
    for t, a in enumerate(accepted):
        d = P.refine_step(st, a, 1.0, entry)
        if d.switched or d.settled_now:
            switches.append(t + 1)
    return switches


def test_planner_exports_every_declared_symbol():
    decl = set(re.findall(r"\b(specsv_[a-z_0-9]+)\s*\(", open(HEADER).read()))
    decl.discard("specsv_last_error")  # named in the header comment, declared in nsa_verify.h
    assert decl == set(P.EXPORTED)
    L = abi.lib()
    for name in decl:
        assert hasattr(L, name), name


def test_bucket_of():  # test_planner.cpp:94-104
    for ctx, b in ((0, 0), (4095, 0), (4096, 1), (5000, 1), (8192, 2), (12288, 3), (16384, 3),
                   (20000, 3)):
        assert P.bucket_of(ctx) == b
    with pytest.raises(abi.SpecsvError):
        P.bucket_of(-1)


def test_precision_classes():  # test_planner.cpp:106-119
    s = P.StrategyTuple(mode=P.EXACT)
    assert P.satisfies(s, P.STRICT) and not P.satisfies(s, P.REUSE_ONLY)
    s.reuse_set = [1]
    assert P.satisfies(s, P.REUSE_ONLY)
    s.mode = P.APPROX
    assert P.satisfies(s, P.APPROX_REUSE)
    s.reuse_set = []
    assert P.satisfies(s, P.APPROX_ONLY)
    with pytest.raises(abi.SpecsvError):
        P.validate_strategy(s, P.STRICT)


def test_strategy_text_round_trip():  # test_planner.cpp:121-131
    s = P.parse_strategy("4,2,BFS,2,exact")
    assert (s.depth, s.width, s.traversal, s.group_size, s.mode) == (4, 2, P.BFS, 2, P.EXACT)
    assert s.to_string() == "4,2,BFS,2,exact"
    for bad in ("4,2,BFS,2", "4,2,XFS,2,exact", "0,2,BFS,2,exact"):
        with pytest.raises(abi.SpecsvError):
            P.parse_strategy(bad)
    assert P.StrategyTuple(2, 2, P.DFS, 4, P.APPROX, [1, 3]).to_string() == "2,2,DFS,4,approx/S=1+3"


def test_profile_offline_192_entries():  # test_planner.cpp:133-191
    cands = default_candidates()
    raw = []
    table = P.profile_offline(lambda s, b, c: fake_eval(s, b, c, raw), cands)
    assert table.stored_strategies() == 4 * 4 * 12
    for b in range(P.NUM_BUCKETS):
        for c in range(P.NUM_CLASSES):
            entry = table.grid(b, c)
            for cand in entry:
                assert P.satisfies(cand.strategy, c)
            for i in range(1, len(entry)):
                assert entry[i - 1].throughput >= entry[i].throughput
    # ranking matches an independent E[A]/E[T] recomputation from the raw log
    for b, c, s, tr in raw:
        thr = (sum(tr.step_accepted) / len(tr.step_accepted)) / (
            sum(tr.step_latency) / len(tr.step_latency))
        for cand in table.grid(b, c):
            if cand.strategy.to_string() == s.to_string():
                assert cand.throughput == pytest.approx(thr, rel=1e-12)
    # missing class candidates raise a configuration error
    only_strict = [s for s in cands if P.satisfies(s, P.STRICT)]
    with pytest.raises(abi.SpecsvError):
        P.profile_offline(fake_eval, only_strict)


def test_preselect_touches_exactly_one_entry():  # test_planner.cpp:193-203
    table = P.profile_offline(fake_eval, default_candidates())
    table.entry_accesses = 0
    best = P.preselect(table, 2, P.REUSE_ONLY)
    assert table.entry_accesses == 1
    assert best.throughput == table.grid(2, P.REUSE_ONLY)[0].throughput
    assert P.satisfies(best.strategy, P.REUSE_ONLY)
    with pytest.raises(abi.SpecsvError):
        P.preselect(P.ProfileTable(), 0, P.STRICT)


def test_guard_switches_at_step_13():  # test_planner.cpp:205-213
    st = P.RefinerState()
    switches = run_trace(st, entry_with_expectations([4.0, 4.0, 4.0]), [2.0] * 32)
    assert switches and switches[0] == 13  # warmup 8 + 5 consecutive sub-threshold steps


def test_guard_no_switch_when_matching():  # test_planner.cpp:215-222
    st = P.RefinerState()
    assert run_trace(st, entry_with_expectations([4.0, 4.0]), [4.0] * 40) == []
    assert st.transitions == 0


def test_guard_two_transitions_then_settle():  # test_planner.cpp:224-238
    st = P.RefinerState()
    switches = run_trace(st, entry_with_expectations([4.0] * 4), [2.0] * 40)
    assert st.transitions == 2 and st.settled
    assert switches == [13, 18, 23]  # warmup does not restart, hysteresis does
    assert st.active_rank <= 2


def test_guard_hysteresis_direction():  # test_planner.cpp:240-258
    noisy = [2.2 if t % 7 < 4 else 4.2 for t in range(64)]

    def events(h):
        st = P.RefinerState(P.GuardConstants(hysteresis=h))
        return len(run_trace(st, entry_with_expectations([4.0] * 6), noisy))

    e3, e5, e8 = events(3), events(5), events(8)
    assert e3 >= e5 >= e8 and e3 > 0


def test_guard_determinism():  # test_planner.cpp:260-272
    rng = Rng(78)
    trace = [1.5 + 2.5 * rng.next_unit() for _ in range(48)]
    entry = entry_with_expectations([4.0, 3.5, 3.0])
    a, b = P.RefinerState(), P.RefinerState()
    assert run_trace(a, entry, trace) == run_trace(b, entry, trace)
    assert (a.active_rank, a.transitions) == (b.active_rank, b.transitions)


def test_guard_transitions_bounded():  # test_planner.cpp:274-285
    rng = Rng(79)
    for _ in range(20):
        st = P.RefinerState()
        run_trace(st, entry_with_expectations([4.0] * 5), [5.0 * rng.next_unit() for _ in range(100)])
        assert st.transitions <= P.MAX_TRANSITIONS


def test_guard_observed_throughput():
    st = P.RefinerState()
    entry = entry_with_expectations([4.0, 4.0])
    for _ in range(3):
        P.refine_step(st, 2.0, 4.0, entry)
    assert st.observed_throughput(0) == pytest.approx(0.5)
    assert st.observed_throughput(1) == 0.0


def layer_stats(unique, constructions, window):
    return {"unique_block_loads": unique, "index_constructions": constructions,
            "window_token_loads": window, "total_requested_loads": unique}


def test_account_step_under_role_plan():  # test_cost_model.cpp:24-40
    L, gamma = 4, 6
    acc = P.account_step([layer_stats(10, gamma, 100)] * L, [2, 3], L)
    assert acc.unique_loads == 40 and acc.window_tokens == 400
    assert acc.constructions == 2 * gamma  # reuse layers construct nothing
    assert acc.launches == 2 * 2 + 2 * 1
    with pytest.raises(abi.SpecsvError):
        P.account_step([layer_stats(10, gamma, 100)] * (L - 1), [2, 3], L)


def test_accounting_strict_and_approx():  # test_cost_model.cpp:42-60
    assert P.account_step([layer_stats(16, 12, 64)] * 8, [], 8).constructions == 12 * 8
    S = list(range(1, 16, 2))
    assert P.account_step([layer_stats(16, 16, 64)] * 16, S, 16).constructions == 16 * 8


def test_estimate_latency_linear_monotone():  # test_cost_model.cpp:62-97
    c = P.CostCoeffs(c_block=2.0, c_index=0.0, c_launch=0.0, c_window=0.0, c_base=5.0)
    a = P.StepAccounting(unique_loads=10)
    assert P.estimate_latency(a, c) == pytest.approx(25.0)
    base = P.CostCoeffs(0.0, 0.0, 0.0, 0.0, 7.0)
    assert P.estimate_latency(a, base) == pytest.approx(7.0)
    b = P.StepAccounting(unique_loads=20)
    assert P.estimate_latency(b, c) - 5.0 == pytest.approx(2 * (P.estimate_latency(a, c) - 5.0))
    for s in range(3, 11):
        x, y = P.StepAccounting(unique_loads=32 - s), P.StepAccounting(unique_loads=32 - s - 1)
        assert P.estimate_latency(y, c) <= P.estimate_latency(x, c)


def test_reuse_never_costs_more():  # test_cost_model.cpp:99-115
    c, L, gamma, prev, S = P.CostCoeffs(), 8, 8, None, []
    for k in range(L):
        if k > 0:
            S.append(k)
        roles = set(S)
        per = [layer_stats(16, 0 if j in roles else gamma, 64) for j in range(L)]
        t = P.estimate_latency(P.account_step(per, S, L), c)
        if prev is not None:
            assert t <= prev
        prev = t


def test_index_share():  # test_cost_model.cpp:117-129
    c = P.CostCoeffs()
    a = P.StepAccounting(unique_loads=10, constructions=10, launches=4, window_tokens=100)
    share = P.index_share(a, c)
    assert 0.0 < share < 1.0
    assert share == pytest.approx(c.c_index * 10.0 / P.estimate_latency(a, c))


def test_fit_recovers_planted_coefficients():  # test_cost_model.cpp:131-170
    rng = Rng(61)
    truth = P.CostCoeffs(c_block=1.5, c_index=4.0, c_launch=0.25, c_window=0.01, c_base=3.0)
    samples = []
    for _ in range(60):
        acc = P.StepAccounting(unique_loads=8 + rng.next_below(64),
                               constructions=rng.next_below(128),
                               launches=8 + rng.next_below(24),
                               window_tokens=100 + rng.next_below(4000))
        samples.append((acc, P.estimate_latency(acc, truth) * (1.0 + 0.02 * (rng.next_unit() - 0.5))))
    fit = P.fit_cost_coeffs(samples)
    assert fit.c_block == pytest.approx(truth.c_block, rel=0.15)
    assert fit.c_index == pytest.approx(truth.c_index, rel=0.15)
    assert fit.c_window == pytest.approx(truth.c_window, rel=0.25)
    fit.validate()
    # anti-correlated data pushes plain least squares negative: clamped
    odd = [(P.StepAccounting(unique_loads=i), 10.0 - 0.1 * i) for i in range(20)]
    P.fit_cost_coeffs(odd).validate()
    with pytest.raises(abi.SpecsvError):
        P.fit_cost_coeffs([])
