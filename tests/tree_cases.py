"""Deterministic draft-tree cases shared by tests/test_draft_tree.py and
tests/golden/make_tree_golden.py: proposers (the reference test's scripted
arithmetic proposer, tests/test_draft_tree.cpp:19-27, and a hashed one with
uneven scores and ties) and the expansion shapes, including C3's
D=6, k=4, budget=32."""
import numpy as np

MASK64 = (1 << 64) - 1


def arithmetic_proposer(step=-0.1):
    def propose(node, token, depth, cum, k):
        return [(token * 10 + 1 + i, step * (i + 1)) for i in range(k)]
    return propose


def _mix(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def hashed_proposer(seed):
    """k distinct tokens with non-increasing scores on a coarse grid (ties
    among siblings and across the frontier exercise the id / seq tie-breaks)."""
    def propose(node, token, depth, cum, k):
        h = _mix(seed * 1000003 + token * 131 + depth)
        scores = sorted((-((_mix(h + i) % 8) / 8.0) for i in range(k)), reverse=True)
        return [((token * 7 + 1 + i + (h % 5)) % 1000003, s) for i, s in enumerate(scores)]
    return propose


# (name, root_token, proposer factory, D, k, budget)
CASES = [
    ("d1k1", 7, lambda: arithmetic_proposer(), 1, 1, None),
    ("d2k2", 7, lambda: arithmetic_proposer(), 2, 2, None),
    ("d3k3", 7, lambda: arithmetic_proposer(), 3, 3, None),
    ("d4k3_b10", 7, lambda: arithmetic_proposer(), 4, 3, 10),
    ("chain4", 7, lambda: arithmetic_proposer(), 4, 1, None),
    ("c3_d6k4_b32", 3, lambda: hashed_proposer(1), 6, 4, 32),
    ("hash_d4k3_b20", 11, lambda: hashed_proposer(2), 4, 3, 20),
    ("hash_d3k4", 5, lambda: hashed_proposer(3), 3, 4, None),
    ("hash_d16k1", 9, lambda: hashed_proposer(4), 16, 1, None),
]


def argmax_for(parent, token, seed):
    """A target argmax per node: with probability 2/3 one of the node's
    children's tokens (so the greedy walk advances), else a token no child holds."""
    rng = np.random.default_rng(seed)
    n = len(parent)
    kids = [[] for _ in range(n)]
    for i in range(1, n):
        kids[int(parent[i])].append(i)
    out = np.zeros(n, np.int32)
    for i in range(n):
        if kids[i] and rng.random() < 2 / 3:
            out[i] = token[kids[i][int(rng.integers(len(kids[i])))]]
        else:
            out[i] = 2_000_000_000 - i
    return out
