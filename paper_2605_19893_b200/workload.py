"""Synthetic Llama-3.1-8B-shaped verify workloads (host side, numpy).

Draws follow the reference's splitmix64 stream (include/specsv/rng.hpp:17-29):
``next_symmetric(a) = float((2 * unit - 1) * a)`` with ``unit = (z >> 11) * 2^-53``.
The generator is vectorised: draw i of a stream seeded with ``s`` is
``mix(s + (i + 1) * 0x9e3779b97f4a7c15)``.

KV is rounded to bf16 (round-to-nearest-even) because the device cache is
bf16; the fp32 upcast of the same bits is what the CPU oracle consumes
(precision plumbing).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix_symmetric(seed: int, a: float, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    unit = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return ((2.0 * unit - 1.0) * a).astype(np.float32)


def splitmix_unit(seed: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (RNE) -> fp32, finite inputs."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 (already bf16-representable) -> uint16 bf16 bit patterns."""
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def chain_tree_mask(gamma: int) -> np.ndarray:
    """Chain draft: row i admits 0..i (tests/test_draft_tree.cpp:115-120)."""
    words = max(1, (gamma + 63) // 64)
    m = np.zeros((max(gamma, 1), words), np.uint64)
    for i in range(gamma):
        for j in range(i + 1):
            m[i, j // 64] |= np.uint64(1) << np.uint64(j % 64)
    return m


def tree_mask_from_parents(parent_slot: list[int]) -> np.ndarray:
    """Ancestor-or-self mask from flat-order parent slots (-1 = root's child),
    the layout build_tree_mask produces (src/draft_tree.cpp:126-141)."""
    gamma = len(parent_slot)
    words = max(1, (gamma + 63) // 64)
    m = np.zeros((max(gamma, 1), words), np.uint64)
    for i in range(gamma):
        j = i
        while j >= 0:
            m[i, j // 64] |= np.uint64(1) << np.uint64(j % 64)
            j = parent_slot[j]
    return m


def depths_from_parents(parent_slot: list[int]) -> list[int]:
    d = []
    for i, p in enumerate(parent_slot):
        d.append(1 if p < 0 else d[p] + 1)
    return d


class LayerInputs:
    """One (request, layer) verify unit: committed KV (bf16-exact fp32), the
    draft rows, queries, gates and positions."""

    def __init__(self, cfg, rows: int, gamma: int, seed: int, parent_slot=None,
                 q_sigma: float | None = None):
        H, dh, Hq = cfg.n_kv_heads, cfg.d_head, cfg.n_q_heads
        self.cfg, self.rows, self.gamma = cfg, rows, gamma
        self.k = bf16_round(splitmix_symmetric(seed * 7 + 1, 1.0, rows * H * dh)).reshape(rows, H, dh)
        self.v = bf16_round(splitmix_symmetric(seed * 7 + 2, 1.0, rows * H * dh)).reshape(rows, H, dh)
        g = max(gamma, 1)
        self.tree_k = bf16_round(splitmix_symmetric(seed * 7 + 3, 1.0, g * H * dh)).reshape(g, H, dh)
        self.tree_v = bf16_round(splitmix_symmetric(seed * 7 + 4, 1.0, g * H * dh)).reshape(g, H, dh)
        nq = 1 + gamma
        if q_sigma is None:
            self.q = splitmix_symmetric(seed * 7 + 5, 1.0, nq * Hq * dh).reshape(nq, Hq, dh)
        else:
            # overlap control: q_i = q_base + sigma * eps_i
            base = splitmix_symmetric(seed * 7 + 5, 1.0, Hq * dh).reshape(1, Hq, dh)
            eps = splitmix_symmetric(seed * 7 + 6, 1.0, nq * Hq * dh).reshape(nq, Hq, dh)
            self.q = (base + np.float32(q_sigma) * eps).astype(np.float32)
        u = splitmix_unit(seed * 7 + 7, nq * Hq * 3)
        self.gates = (0.2 + 0.6 * u).astype(np.float32).reshape(nq, Hq, 3)
        if parent_slot is None:
            parent_slot = [i - 1 for i in range(gamma)]  # chain
        self.parent_slot = parent_slot
        depths = depths_from_parents(parent_slot) if gamma else []
        self.pos = np.array([rows - 1] + [rows - 1 + dd for dd in depths], np.int64)
        self.tree_mask = tree_mask_from_parents(parent_slot) if gamma else np.zeros((1, 1), np.uint64)
        pe = splitmix_symmetric(seed * 7 + 8, 0.1, cfg.l * dh).reshape(cfg.l, dh)
        self.pos_embed = pe
