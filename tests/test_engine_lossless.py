"""End-to-end losslessness (the reference's SPEC acceptance
1): with exact coarsening, speculative decoding through this repo's verify
path emits exactly the tokens autoregressive decoding emits under the same
strategy (same reuse schedule), from the same synthetic prefilled context.
The engine (paper_2605_19893_b200/engine.py) mirrors run_target_pass and
Engine::step (engine.cpp:107-560)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2605_19893_b200 import engine as E  # noqa: E402
from paper_2605_19893_b200 import tree as T  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("traversal,reuse", [(T.BFS, ()), (T.DFS, (1, 3))])
def test_speculative_equals_autoregressive(traversal, reuse):
    spec = E.ToyModelSpec()
    n_new = 24
    strat = E.Strategy(depth=4, width=2, budget=8, traversal=traversal, group_size=4,
                       reuse_set=reuse)
    ar = E.Engine(spec, prompt_rows=3000, max_context=3200)
    want = ar.generate(n_new, strat, autoregressive=True)
    sp = E.Engine(spec, prompt_rows=3000, max_context=3200)
    got, accepted = [], []
    start = len(sp.tokens)
    while len(sp.tokens) - start < n_new:
        out = sp.step(strat)
        accepted.append(out.accepted)
    got = sp.tokens[start:start + n_new]
    assert got == want
    # the tree proposer is accepted sometimes, so more than one token per step on average
    assert sum(accepted) > len(accepted)
    # the caches agree row for row where both committed the same tokens
    assert sp.caches[0].rows >= 3000 + n_new - 1


@pytest.mark.parametrize("seed", list(range(20)))
def test_lossless_spec_scale(seed):
    """SPEC.md:557's scale: 20 seeds x 128 generated tokens, each seed a
    different toy model, prefilled context and strategy (BFS / DFS, with and
    without reuse layers, tree shape): speculative == autoregressive."""
    spec = E.ToyModelSpec(seed=100 + seed)
    strat = E.Strategy(depth=2 + seed % 4, width=1 + seed % 3, budget=4 + 2 * (seed % 5),
                       traversal=T.BFS if seed % 2 == 0 else T.DFS, group_size=1 + seed % 4,
                       reuse_set=() if seed % 3 == 0 else ((1, 3) if seed % 3 == 1 else (2,)))
    n_new = 128
    ar = E.Engine(spec, prompt_rows=1500 + 37 * seed, max_context=1900 + 37 * seed, seed=seed)
    want = ar.generate(n_new, strat, autoregressive=True)
    sp = E.Engine(spec, prompt_rows=1500 + 37 * seed, max_context=1900 + 37 * seed, seed=seed)
    start = len(sp.tokens)
    while len(sp.tokens) - start < n_new:
        sp.step(strat)
    assert sp.tokens[start:start + n_new] == want
