"""Generate golden vectors for the verify hot path by running the REFERENCE
(oracle/_ref/libspecsv_ref.so, compiled in place from /root/reference/proj/src)
on deterministic synthetic inputs.  Inputs are NOT stored: they are
regenerated bit-exactly from the seed by paper_2605_19893_b200.workload
(splitmix64, rng.hpp:17-29).  Stored: pooled-cache digests, selected
indices, gated outputs and LoadStats.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2605_19893_b200.workload import LayerInputs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, cfg, rows, gamma, seed, parents, mode, C)
def cases():
    small = O.small_config()
    llama = O.llama_config(n_layers=4)
    tree8 = [-1, -1, 0, 0, 1, 2, 2, 4]          # 2 roots' children, depth <= 4
    return [
        ("small_chain_exact", small, 160, 4, 1, None, O.MODE_EXACT, 2),
        ("small_chain_approx", small, 160, 4, 2, None, O.MODE_APPROX, 2),
        ("small_tree_exact", small, 200, 8, 3, tree8, O.MODE_EXACT, 4),
        ("small_tree_approx", small, 200, 8, 4, tree8, O.MODE_APPROX, 4),
        ("small_short_ctx", small, 20, 3, 5, None, O.MODE_EXACT, 1),
        ("llama_c1_chain4", llama, 4096, 4, 6, None, O.MODE_EXACT, 4),
        ("llama_2k_chain8_approx", llama, 2048 + 37, 8, 7, None, O.MODE_APPROX, 4),
        ("llama_1k_tree8", llama, 1000, 8, 8, tree8, O.MODE_EXACT, 2),
    ]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_case(lib, name, cfg, rows, gamma, seed, parents, mode, C):
    x = LayerInputs(cfg, rows, gamma, seed, parent_slot=parents)
    ck, cv = lib.build_compressed(cfg, x.k, x.v, rows, x.pos_embed)
    gates = x.gates.astype(np.float64)
    ref = lib.verify_layer(cfg, x.k, x.v, ck, cv, x.q, x.pos, gates, x.tree_k, x.tree_v,
                           x.tree_mask, C, mode, O.ROLE_REFRESH)
    # reuse layer: a second layer's KV with the refresh layer's sets inherited
    y = LayerInputs(cfg, rows, gamma, seed + 1000, parent_slot=parents)
    ck2, cv2 = lib.build_compressed(cfg, y.k, y.v, rows, y.pos_embed)
    reuse = lib.verify_layer(cfg, y.k, y.v, ck2, cv2, y.q, x.pos, y.gates.astype(np.float64),
                             y.tree_k, y.tree_v, x.tree_mask, C, mode, O.ROLE_REUSE,
                             idx=ref["idx"], idx_count=ref["idx_count"],
                             idx_forced=ref["idx_forced"])
    return dict(
        meta=json.dumps(dict(name=name, cfg=cfg.__dict__, rows=rows, gamma=gamma, seed=seed,
                             parents=parents, mode=mode, C=C)),
        ck_sha=digest(ck), cv_sha=digest(cv), ck2_sha=digest(ck2), cv2_sha=digest(cv2),
        refresh_out=ref["out"], refresh_idx=ref["idx"], refresh_cnt=ref["idx_count"],
        refresh_forced=ref["idx_forced"], refresh_stats=json.dumps(ref["stats"]),
        reuse_out=reuse["out"], reuse_idx=reuse["idx"], reuse_cnt=reuse["idx_count"],
        reuse_stats=json.dumps(reuse["stats"]),
    )


def main():
    lib = O.load("ref")
    assert lib.name == "reference"
    for c in cases():
        res = run_case(lib, *c)
        np.savez_compressed(os.path.join(HERE, c[0] + ".npz"), **res)
        print("wrote", c[0])


if __name__ == "__main__":
    main()
