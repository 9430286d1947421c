"""Desk-scale speculative-decoding engine around the verify path (SURVEY §8f
row 4): the target layer stack of the reference's toy model with this
repo's NSA verify in every layer, a tree proposer, greedy acceptance and the
commit of accepted rows -- used to check end-to-end losslessness (exact mode:
speculative decoding emits exactly the tokens autoregressive decoding does
under the same strategy, the reference's SPEC acceptance 1).

Mirrors (paths relative to /root/reference/proj):
  ToyModelSpec / ToyModel            include/specsv/model/toy_model.hpp:20-64
  run_target_pass (per layer:        src/engine.cpp:107-280
    rmsnorm, q/k/v projections, root row appended before attention, gates
    = sigmoid(w_gate . q_h), compressed extension, routing / reuse, verify,
    wo + residual, ReLU MLP + residual)
  readout_logits (W_out . rmsnorm(h) + bigram[token])   src/engine.cpp:282-299
  Engine::step (expand, flatten, verify, greedy accept, commit)
                                     src/engine.cpp:471-560

The layer GEMMs and norms run in PyTorch: they are the model around the hot
path, not the path (the reference runs them as scalar loops).  Everything
on the verify path -- routing, attention, compressed-block pooling, tree
flattening, greedy accept, the commit -- goes through the C-ABI.  The
committed context is a synthetic prefilled cache (random K/V rows), shared
by both decoding modes; the draft proposer is the model's own bigram table
(draft quality changes the acceptance length, never the emitted tokens).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import tree as T
from . import verify as V


@dataclass
class ToyModelSpec:
    seed: int = 1
    n_layers: int = 4
    vocab: int = 512
    mlp_mult: int = 2
    bigram_scale: float = 4.0
    nsa: V.NsaConfig = field(default_factory=lambda: V.NsaConfig(
        l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=8, n_kv_heads=2, d_head=128, n_layers=4,
        routing_lag=16))

    @property
    def hidden(self) -> int:
        return self.nsa.n_q_heads * self.nsa.d_head


@dataclass
class Strategy:
    """The StrategyTuple fields the step uses (plan/strategy.hpp:14-45)."""
    depth: int = 4
    width: int = 2
    budget: int = 8
    traversal: int = T.BFS
    group_size: int = 4
    mode: int = V.MODE_EXACT
    reuse_set: tuple = ()


@dataclass
class StepOutcome:
    gamma: int
    accepted: int            # A_t, bonus included
    committed: List[int]     # accepted tokens + bonus


class ToyModel:
    """Seeded uniform weights with the reference's scales (toy_model.cpp:37-107)."""

    def __init__(self, spec: ToyModelSpec, device="cuda"):
        self.spec = spec
        g = torch.Generator(device="cpu")
        g.manual_seed(spec.seed)
        h, c = spec.hidden, spec.nsa
        kvdim, mlp = c.n_kv_heads * c.d_head, spec.mlp_mult * spec.hidden

        def u(*shape, scale):
            return ((torch.rand(*shape, generator=g) * 2 - 1) * scale).to(device)

        s_h, s_mlp = 1.0 / h ** 0.5, 1.0 / mlp ** 0.5
        self.embedding = u(spec.vocab, h, scale=0.5)
        self.key_pos_embed = u(c.l, c.d_head, scale=0.1)
        self.layers = [dict(wq=u(h, h, scale=s_h), wk=u(kvdim, h, scale=s_h),
                            wv=u(kvdim, h, scale=s_h), wo=u(h, h, scale=s_h),
                            w_gate=u(3, c.d_head, scale=1.0 / c.d_head ** 0.5),
                            mlp_in=u(mlp, h, scale=s_h), mlp_out=u(h, mlp, scale=s_mlp))
                       for _ in range(spec.n_layers)]
        self.w_out = u(spec.vocab, h, scale=s_h)
        self.bigram = u(spec.vocab, spec.vocab, scale=spec.bigram_scale)
        idx = torch.arange(h, device=device)
        self.freq = torch.pow(10000.0, -(idx // 2 * 2).double() / h)

    def embed(self, tokens: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        """token embedding + 0.1 x sinusoidal position (toy_model.cpp:109-120)."""
        ang = pos.double()[:, None] * self.freq[None, :]
        p = torch.where(torch.arange(self.spec.hidden, device=ang.device) % 2 == 0, ang.sin(), ang.cos())
        return self.embedding[tokens] + 0.1 * p.float()


def _rmsnorm(x: torch.Tensor) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + 1e-6)


class Engine:
    """One request's target model + caches; step() is Engine::step."""

    def __init__(self, spec: ToyModelSpec, prompt_rows: int, max_context: int, seed: int = 11,
                 device="cuda"):
        self.spec, self.cfg, self.dev = spec, spec.nsa, device
        self.model = ToyModel(spec, device)
        c = self.cfg
        self.caches = []
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        for _ in range(spec.n_layers):  # synthetic prefilled context
            kv = V.LayerCache(c, max_context, device=device)
            kv.append(((torch.rand(prompt_rows, c.n_kv_heads, c.d_head, generator=g, device=device) * 2 - 1)
                       * 0.5).bfloat16(),
                      ((torch.rand(prompt_rows, c.n_kv_heads, c.d_head, generator=g, device=device) * 2 - 1)
                       * 0.5).bfloat16())
            kv.extend_compressed(self.model.key_pos_embed)
            self.caches.append(kv)
        self.tokens = [int(torch.randint(spec.vocab, (1,), generator=g, device=device).item())]
        self.ws = V.Workspace(c, 1 + 64, max_context, device=device)

    # ---- the draft side: bigram top-k proposer ------------------------------
    def _propose(self, node, token, depth, cum, k):
        row = self.model.bigram[token]
        top = torch.topk(row, k)
        return [T.TokenScore(int(t), float(s)) for s, t in zip(top.values.tolist(), top.indices.tolist())]

    def _readout(self, hidden: torch.Tensor, tokens: torch.Tensor) -> torch.Tensor:
        return _rmsnorm(hidden) @ self.model.w_out.T + self.model.bigram[tokens]

    def _target_pass(self, toks: List[int], pos: np.ndarray, tmask: np.ndarray, strat: Strategy):
        """run_target_pass: query 0 is the pending root (its row is committed
        before attention), the rest are tree queries in flat order."""
        c, dev = self.cfg, self.dev
        nq = len(toks)
        gamma = nq - 1
        roles, source = V.resolve_layer_roles(list(strat.reuse_set), self.spec.n_layers)
        tok_t = torch.tensor(toks, device=dev)
        hidden = self.model.embed(tok_t, torch.tensor(pos, device=dev))
        sets = [V.IndexSets.empty(nq, c.n, dev) for _ in range(self.spec.n_layers)]
        scratch = []
        Hq, Hkv, dh = c.n_q_heads, c.n_kv_heads, c.d_head
        for j, lw in enumerate(self.model.layers):
            xn = _rmsnorm(hidden)
            q = xn @ lw["wq"].T
            k = (xn @ lw["wk"].T).view(nq, Hkv, dh).bfloat16()
            v = (xn @ lw["wv"].T).view(nq, Hkv, dh).bfloat16()
            kv = self.caches[j]
            kv.append(k[:1], v[:1])  # the root's row, before any attention
            kv.extend_compressed(self.model.key_pos_embed)
            tk = k[1:].contiguous() if gamma else None
            tv = v[1:].contiguous() if gamma else None
            scratch.append((tk, tv))
            qh = q.view(nq, Hq, dh)
            gates = torch.sigmoid(torch.einsum("qhd,bd->qhb", qh, lw["w_gate"])).contiguous()
            batch = V.DraftBatch(pos=pos, tree_mask=tmask, q=qh.contiguous(), gates=gates,
                                 tree_k=tk, tree_v=tv)
            out = torch.zeros(nq, Hq, dh, device=dev)
            s = sets[j] if roles[j] == V.ROLE_REFRESH else sets[int(source[j])]
            V.nsa_verify(c, kv, batch, s, out, self.ws, strat.group_size, strat.mode, int(roles[j]))
            hidden = hidden + out.view(nq, -1) @ lw["wo"].T
            hidden = hidden + torch.relu(_rmsnorm(hidden) @ lw["mlp_in"].T) @ lw["mlp_out"].T
        argmax = self._readout(hidden, tok_t).argmax(dim=-1)
        return argmax.tolist(), scratch

    def step(self, strat: Strategy, autoregressive: bool = False) -> StepOutcome:
        """Engine::step (engine.cpp:471-560)."""
        c = self.caches[0].rows + 1  # committed tokens, the pending root included (its row comes in the pass)
        if autoregressive:
            tree = T.DraftTree.from_nodes([(-1, self.tokens[-1], 0.0)])
            flat = T.FlatBatch(T.BFS, np.zeros(0, np.int64), np.zeros(0, np.int64),
                               np.zeros((0, 1), np.uint64), 0)
        else:
            tree = T.expand_draft_tree(self.tokens[-1], self._propose, strat.depth, strat.width,
                                       strat.budget)
            flat = T.flatten_tree(tree, strat.traversal, c)
        toks = [self.tokens[-1]] + [int(tree.token[n]) for n in flat.order]
        pos = np.array([c - 1] + flat.positions.tolist(), np.int64)
        tmask = flat.mask if flat.gamma else np.zeros((1, 1), np.uint64)
        am, scratch = self._target_pass(toks, pos, tmask, strat)
        argmax = np.zeros(tree.n_nodes, np.int32)  # per node: query 0 = root, 1 + i = order[i]
        argmax[0] = am[0]
        for i, n in enumerate(flat.order):
            argmax[int(n)] = am[1 + i]
        vr = T.greedy_verify(tree, argmax)
        if vr.accepted_nodes:
            slot = {int(n): i for i, n in enumerate(flat.order)}
            T.commit_accepted(self.cfg, self.caches, [s[0] for s in scratch], [s[1] for s in scratch],
                              [slot[n] for n in vr.accepted_nodes], pos_embed=self.model.key_pos_embed)
        self.tokens += vr.accepted_tokens + [vr.bonus_token]
        return StepOutcome(flat.gamma, vr.accepted_count, vr.accepted_tokens + [vr.bonus_token])

    def generate(self, n_tokens: int, strat: Strategy, autoregressive: bool = False) -> List[int]:
        start = len(self.tokens)
        while len(self.tokens) - start < n_tokens:
            self.step(strat, autoregressive)
        return self.tokens[start:start + n_tokens]
