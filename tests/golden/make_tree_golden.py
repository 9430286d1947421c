"""Generate golden vectors for the draft-tree utilities by running the
REFERENCE (proj/src/draft_tree.cpp via oracle/_ref/libspecsv_ref.so and
oracle/ref_tree_shim.cpp) on the deterministic cases of tests/tree_cases.py:
the expanded trees, their BFS/DFS flattening (order, positions, unpacked
mask) and greedy acceptance under seeded target argmaxes.

    python tests/golden/make_tree_golden.py     # rewrites tests/golden/draft_trees.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.tree_cases import CASES, argmax_for  # noqa: E402

COMMITTED = 65536


def main():
    ref = O.RefTree()
    out = {}
    for ci, (name, root, mk, D, k, budget) in enumerate(CASES):
        rc, (parent, token, depth, score, cum) = ref.expand(root, mk(), D, k, budget)
        assert rc == 0, name
        pre = f"{name}/"
        out[pre + "parent"], out[pre + "token"], out[pre + "depth"] = parent, token, depth
        out[pre + "score"], out[pre + "cum"] = score, cum
        for trav in (0, 1):
            order, pos, mask = ref.flatten(parent, token, depth, score, trav, COMMITTED)
            out[pre + f"order{trav}"], out[pre + f"pos{trav}"] = order, pos
            out[pre + f"mask{trav}"] = mask.astype(np.uint8)
        for s in range(3):
            am = argmax_for(parent, token, 100 * ci + s)
            rc, nodes, toks, bonus = ref.greedy(parent, token, depth, score, am)
            assert rc == 0
            out[pre + f"argmax{s}"] = am
            out[pre + f"acc_nodes{s}"] = np.array(nodes, np.int64)
            out[pre + f"acc_tokens{s}"] = np.array(toks, np.int32)
            out[pre + f"bonus{s}"] = np.array([bonus], np.int32)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "draft_trees.npz")
    np.savez_compressed(path, **out)
    print(path, len(CASES), "cases")


if __name__ == "__main__":
    main()
