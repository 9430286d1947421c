"""Shared helpers for the GPU parity tests: build one verify unit on the device
from a deterministic LayerInputs, run the sm_100a path through the C-ABI, and
run the CPU oracle on the identical (bf16-exact) inputs.

Precision plumbing: K/V are bf16 on the device; the oracle gets
their fp32 upcast.  The compressed values are stored bf16 on the device, so
the oracle is fed the same bf16-rounded pooled values (ck stays fp32 and is
bit-exact)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O
from paper_2605_19893_b200 import verify as V
from paper_2605_19893_b200.workload import LayerInputs, bf16_round

TOL = 2e-3  # north-star output tolerance (fp32 accumulation over bf16 KV)


def to_dev_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


class DeviceCase:
    def __init__(self, cfg: O.NsaConfig, x: LayerInputs):
        self.cfg, self.x = cfg, x
        self.vcfg = V.NsaConfig(**cfg.__dict__)
        rows = x.k.shape[0]
        self.cache = V.LayerCache(self.vcfg, rows)
        self.cache.append(to_dev_bf16(x.k), to_dev_bf16(x.v))
        self.pe = torch.from_numpy(x.pos_embed).cuda()
        self.cache.extend_compressed(self.pe)
        g = x.gamma
        self.batch = V.DraftBatch(
            pos=x.pos, tree_mask=x.tree_mask,
            q=torch.from_numpy(x.q).cuda(), gates=torch.from_numpy(x.gates).cuda(),
            tree_k=to_dev_bf16(x.tree_k[:max(g, 1)]) if g else None,
            tree_v=to_dev_bf16(x.tree_v[:max(g, 1)]) if g else None)
        self.ws = V.Workspace(self.vcfg, 1 + g, rows)
        self.nq = 1 + g

    def run(self, group_size=4, mode=V.MODE_EXACT, role=V.ROLE_REFRESH, sets=None):
        sets = sets or V.IndexSets.empty(self.nq, self.cfg.n)
        out = torch.zeros(self.nq, self.cfg.n_q_heads, self.cfg.d_head, device="cuda")
        V.nsa_verify(self.vcfg, self.cache, self.batch, sets, out, self.ws, group_size, mode, role)
        torch.cuda.synchronize()
        return out.cpu().numpy().astype(np.float64), sets

    def oracle_cache(self, lib):
        ck, cv = lib.build_compressed(self.cfg, self.x.k, self.x.v, self.x.k.shape[0],
                                      self.x.pos_embed)
        return ck, bf16_round(cv)

    def oracle(self, lib, group_size=4, mode=O.MODE_EXACT, role=O.ROLE_REFRESH, idx=None,
               idx_count=None, idx_forced=None):
        ck, cv = self.oracle_cache(lib)
        x = self.x
        g = x.gamma
        return lib.verify_layer(self.cfg, x.k, x.v, ck, cv, x.q, x.pos,
                                x.gates.astype(np.float64), x.tree_k[:max(g, 1)],
                                x.tree_v[:max(g, 1)], x.tree_mask, group_size, mode, role,
                                idx=idx, idx_count=idx_count, idx_forced=idx_forced)


def rel_errors(got, ref):
    """per (query, head): ||o_gpu - o_ref||_inf / max(||o_ref||_inf, 1e-6); global rel L2."""
    d = np.abs(got - ref).max(-1)
    n = np.maximum(np.abs(ref).max(-1), 1e-6)
    per = d / n
    l2 = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-12)
    return float(per.max()), float(l2)


def sets_to_numpy(sets: V.IndexSets):
    return (sets.idx.cpu().numpy().astype(np.int64), sets.count.cpu().numpy().astype(np.int64),
            sets.forced.cpu().numpy().astype(np.int64) & 0xFFFFFFFF)


def forced_matrix(forced_bits, n):
    return np.array([[(int(f) >> i) & 1 for i in range(n)] for f in forced_bits], np.uint8)


def boundary_gap(lib, cfg, q, ck, pos):
    """Relative gap between the n-th and (n+1)-th non-forced reference scores."""
    vis = cfg.routing_visible_len(int(pos))
    s = lib.selection_scores(cfg, q, ck, vis)
    avail = s.size
    forced = {0, avail - 2, avail - 1} if avail > 2 else set(range(avail))
    rest = np.sort(np.array([s[b] for b in range(avail) if b not in forced]))[::-1]
    k = cfg.n - len(forced)
    if k <= 0 or k >= rest.size:
        return np.inf
    return float((rest[k - 1] - rest[k]) / max(rest[k - 1], 1e-300))


def diff_within_near_tie(lib, cfg, q, ck, pos, got, want, near_tie):
    """True when every block in the symmetric difference of two index sets
    has a reference score within `near_tie` (relative) of the Top-n boundary
    score (the n-th best non-forced score): the sets differ only by a flip at
    a near-tie, nothing else (contract P2)."""
    vis = cfg.routing_visible_len(int(pos))
    s = lib.selection_scores(cfg, q, ck, vis)
    avail = s.size
    forced = {0, avail - 2, avail - 1} if avail > 2 else set(range(avail))
    rest = np.sort(np.array([s[b] for b in range(avail) if b not in forced]))[::-1]
    k = cfg.n - len(forced)
    if k <= 0 or k >= rest.size:
        return False
    sb = rest[k - 1]
    diff = set(int(b) for b in got) ^ set(int(b) for b in want)
    return all(b < avail and abs(s[b] - sb) <= near_tie * max(abs(sb), 1e-300) for b in diff)
