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
