#!/usr/bin/env python3
"""Benchmark of the sparse speculative-verification hot path on B200.

Workloads (BASELINE.json configs), Llama-3.1-8B-shaped NSA
(32 q / 8 KV heads, d_head 128, l=32, d=16, l_sel=64, n=16, w=512, lag 16),
8-token chain draft, bf16 KV, EXACT grouping (C=4) with the reference's "alt"
refresh/reuse schedule (layers 1,3,.. reuse the preceding layer's sets):

  C2 (default at 1 GPU; configs[1], the metric's config): 64K committed
     context, one request per GPU, one verify pass over L=32 DISTINCT layer
     caches per step (one C-ABI verify call per layer, like run_target_pass).
     At N GPUs (--workload c2) every rank runs its own request: weak scaling.
  C4 (default at N>1 GPUs; configs[3]): 128K context, 64 requests in total,
     4 layer caches per request, sharded over the ranks by request (64/N each,
     one batched verify call per layer over a rank's requests); with fewer
     requests than ranks (--total-requests) a request is split by KV-head
     group (routing replicated, sharding.shard_plan).  Strong scaling: the
     total work is fixed.

A step touches GBs of KV (>> the 126 MB L2), so successive steps never hit L2
on the same layer.  The step is captured once in a CUDA graph and replayed.

metric: verified query-tokens/s = (requests x (1 + gamma)) / seconds per step
(whole job over all GPUs, max over ranks of the device time).  `e2e` runs
real steps through the public API: every step copies its inputs host->device
(pinned), re-issues every layer's C-ABI verify call with the positions and
committed rows of THAT step (eager: the host work of each call is inside the
timed region), commits the accepted draft rows (specsv_commit_rows +
compressed-block append) so the context grows, and reads the last layer's
output back.

`--gpus N` without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL; only timing gathers and barriers cross ranks).

--impl reference: the reference's own CPU implementation (oracle/_ref, the
reference compiled from its sources) on this host's cores, same workload,
rank 0 only.
--dry-run: the multi-rank orchestration (launch, process group, shard plan,
barrier, max-over-ranks timing, JSON line) with the GPU step replaced by a
CPU stand-in -- the gloo CPU test drives this path.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "query-tokens/s"


def metric_for(ctx: int, gamma: int) -> str:
    # the C2 default reproduces BASELINE.json's metric string exactly
    return (f"verified query-tokens/s at {ctx // 1024}K ctx, {gamma}-tok draft; "
            "achieved HBM GB/s vs peak")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c2", "c4"],
                    help="auto: C2 at 1 GPU, C4 at N > 1")
    ap.add_argument("--ctx", type=int, default=0, help="override the workload's context")
    ap.add_argument("--gamma", type=int, default=8)
    ap.add_argument("--layers", type=int, default=0, help="override the workload's layer caches")
    ap.add_argument("--mode", default="exact", choices=["exact", "approx"])
    ap.add_argument("--group", type=int, default=4)
    ap.add_argument("--schedule", default="alt")
    ap.add_argument("--requests", type=int, default=0,
                    help="C2: requests per GPU (default 1)")
    ap.add_argument("--total-requests", type=int, default=0,
                    help="C4: requests over all GPUs (default 64)")
    ap.add_argument("--accept", type=int, default=4,
                    help="e2e: draft rows accepted (and committed) per step")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-decode-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    return ap.parse_args(argv)


def resolve_workload(a, world: int):
    """Fill the workload's shape into `a` (explicit flags win)."""
    w = a.workload if a.workload != "auto" else ("c2" if world == 1 else "c4")
    a.workload = w
    if w == "c2":
        a.ctx = a.ctx or 65536
        a.layers = a.layers or 32
        per_gpu = a.requests or 1
        a.total_requests = a.total_requests or per_gpu * world  # weak: fixed per-GPU work
        a.scaling = "weak"
    else:
        a.ctx = a.ctx or 131072
        a.layers = a.layers or 4
        a.total_requests = a.total_requests or 64  # strong: fixed total work
        a.scaling = "strong"
    return a


def reuse_set(schedule: str, L: int):
    if schedule in ("", "none"):
        return []
    if schedule == "alt":
        return list(range(1, L, 2))
    return [int(x) for x in schedule.split(",") if x]


def llama_cfg(L):
    from paper_2605_19893_b200.verify import NsaConfig
    return NsaConfig(l=32, d=16, l_sel=64, n=16, w=512, n_q_heads=32, n_kv_heads=8, d_head=128,
                     n_layers=L, routing_lag=16)


def parallelism(a, world: int) -> str:
    if world == 1:
        return "single GPU"
    if a.total_requests >= world:
        return f"request sharding x{world} (no collective on the data path)"
    return (f"request + KV-head-group sharding x{world} ({a.total_requests} requests, routing "
            "replicated per head group, no collective on the data path)")


def workload_config(a, world: int):
    """Identical for both arms (the driver compares the dicts)."""
    name = a.workload.upper()
    per = a.total_requests / world
    return {"workload": f"{name}: Llama-3.1-8B-shaped NSA verify, {a.ctx // 1024}K ctx, "
                        f"{a.gamma}-token chain draft, bf16 KV, {a.layers} layer caches, "
                        f"{a.total_requests} request(s) over {world} GPU(s)",
            "ctx": a.ctx, "draft": "chain", "gamma": a.gamma, "layers": a.layers,
            "total_requests": a.total_requests, "requests_per_gpu": per, "mode": a.mode,
            "group_size": a.group, "schedule": a.schedule, "heads": "32q/8kv", "d_head": 128,
            "nsa": "l=32 d=16 l_sel=64 n=16 w=512 lag=16", "parallelism": parallelism(a, world),
            "l2": "inputs larger than L2 (each step streams every request-layer cache once: GBs, "
                  "L2 is 126 MB)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(a, argv) -> int:
    """--gpus N outside torchrun: one process per GPU under torch.distributed.run
    (rendezvous on 127.0.0.1); rank 0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__), *argv]
    return subprocess.run(cmd).returncode


# --------------------------------------------------------------------------- CPU
class CpuReference:
    """The reference (oracle/_ref: the reference's own C++ compiled in place) on
    this host: independent (layer, request) verify units on host threads
    (SPEC.md:138 allows concurrent queries/layers)."""

    def __init__(self, a, threads: int):
        from oracle import oracle as O
        from paper_2605_19893_b200.workload import LayerInputs
        self.O, self.a, self.threads = O, a, threads
        self.kind = "reference" if O.ref_available() else "port"
        self.lib = O.load("ref" if self.kind == "reference" else "oracle")
        self.cfg = O.llama_config(a.layers)
        self.mode = O.MODE_EXACT if a.mode == "exact" else O.MODE_APPROX
        self.units = []
        for u in range(2):
            x = LayerInputs(self.cfg, a.ctx, a.gamma, 500 + u)
            ck, cv = self.lib.build_compressed(self.cfg, x.k, x.v, a.ctx, x.pos_embed)
            self.units.append((x, ck, cv))
        x0, ck0, cv0 = self.units[0]
        self.seed_sets = self.lib.verify_layer(
            self.cfg, x0.k, x0.v, ck0, cv0, x0.q, x0.pos, x0.gates.astype(np.float64), x0.tree_k,
            x0.tree_v, x0.tree_mask, a.group, self.mode, O.ROLE_REFRESH)
        self.n_reuse = len(reuse_set(a.schedule, a.layers))

    def describe(self):
        try:
            dispatch = self.lib.name
        except Exception:  # noqa: BLE001 -- the port has no dispatch slot
            dispatch = "n/a"
        return {"cpu_model": cpu_model(), "kernel_dispatch": dispatch,
                "SPECSV_KERNEL": os.environ.get("SPECSV_KERNEL", "(unset: avx2 when available)")}

    def measure(self, seconds: float):
        """query-tokens/s for full L-layer steps (schedule's refresh/reuse mix),
        all threads, plus a description of the bounded sample."""
        O, a = self.O, self.a
        times = {O.ROLE_REFRESH: [], O.ROLE_REUSE: []}
        done = [0] * self.threads
        stop = time.time() + seconds

        def worker(tid):
            k = 0
            while k < 2 or time.time() < stop:
                role = O.ROLE_REUSE if (k % 2 == 1 and self.n_reuse > 0) else O.ROLE_REFRESH
                x, ck, cv = self.units[(tid + k) % 2]
                kw = {}
                if role == O.ROLE_REUSE:
                    kw = dict(idx=self.seed_sets["idx"], idx_count=self.seed_sets["idx_count"],
                              idx_forced=self.seed_sets["idx_forced"])
                t0 = time.time()
                self.lib.verify_layer(self.cfg, x.k, x.v, ck, cv, x.q, x.pos,
                                      x.gates.astype(np.float64), x.tree_k, x.tree_v,
                                      x.tree_mask, a.group, self.mode, role, **kw)
                times[role].append(time.time() - t0)
                done[tid] += 1
                k += 1

        t0 = time.time()
        ths = [threading.Thread(target=worker, args=(i,)) for i in range(self.threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        el = time.time() - t0
        tr = float(np.mean(times[O.ROLE_REFRESH]))
        tu = float(np.mean(times[O.ROLE_REUSE])) if times[O.ROLE_REUSE] else tr
        per_step_thread_s = (a.layers - self.n_reuse) * tr + self.n_reuse * tu
        rate = self.threads * (1 + a.gamma) / per_step_thread_s
        sample = (f"{sum(done)} single-layer verify calls of the workload ({a.ctx // 1024}K ctx, "
                  f"gamma={a.gamma}, {a.mode} C={a.group}; mean refresh {tr * 1e3:.0f} ms, reuse "
                  f"{tu * 1e3:.0f} ms per call per thread) on {self.threads} threads in {el:.1f} s, "
                  f"scaled to {a.layers}-layer steps ({a.layers - self.n_reuse} refresh + "
                  f"{self.n_reuse} reuse layers) of one request")
        return rate, sample


def run_reference_arm(a, world: int, rank: int):
    if rank != 0:
        return
    threads = a.cpu_threads or os.cpu_count() or 1
    ref = CpuReference(a, threads)
    per_step = max(1.0, min(5.0, 150.0 / max(1, a.steps + a.warmup)))
    vals, sample = [], ""
    for s_ in range(a.warmup + a.steps):
        rate, smp = ref.measure(per_step if s_ >= a.warmup else 0.0)
        if s_ >= a.warmup:
            vals.append(rate)
            sample = sample or smp
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": metric_for(a.ctx, a.gamma), "value": v, "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * a.total_requests * (1 + a.gamma) / v,
            "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (splitmix64 U[-1,1] KV/q, bf16-rounded)",
            "config": workload_config(a, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": ref.kind,
                             "sample": sample, **ref.describe()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU
class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = f"/tmp/specsv_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except OSError:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def ncu_traffic(workload: str, n_req_launch: int):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture of the SAME workload (profiles/), or None."""
    name = "r02_attend_ncu_summary.json" if n_req_launch == 1 else "r02_attend_batch_c4_ncu_summary.json"
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", name)))
    except (OSError, ValueError):
        return None, None
    if prof.get("workload", workload.upper()) != workload.upper():
        return None, name
    if int(prof.get("requests_per_launch", 1 if n_req_launch == 1 else 8)) != n_req_launch:
        return None, name
    return prof.get("dram_bytes_per_launch"), name


def run_dry(a, world: int, rank: int):
    """The orchestration of run_ours with a CPU stand-in for the GPU step."""
    import torch.distributed as dist

    from paper_2605_19893_b200 import sharding
    if world > 1:
        dist.init_process_group("gloo")
    shards = sharding.shard_plan(a.total_requests, world, rank, 8)
    nq = 1 + a.gamma
    units = sum(s.fraction for s in shards) * nq
    ms = 1.0 + 0.25 * rank  # stand-in device time: the slowest rank sets the step
    value, ms_max = sharding.job_throughput(units, ms)
    plan = [[(s.request, s.head_begin, s.head_count) for s in shards]]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, plan[0])
        plan = gathered
    if rank == 0:
        line = {"metric": metric_for(a.ctx, a.gamma), "value": value, "unit": UNIT,
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max,
                "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
                "dtype": "bf16", "data": "dry run (no GPU): CPU stand-in step",
                "config": workload_config(a, world), "dry_run": True, "shard_plan": plan}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(a, world: int, rank: int, local: int):
    import torch
    import torch.distributed as dist

    from paper_2605_19893_b200 import sharding
    from paper_2605_19893_b200 import tree as TR
    from paper_2605_19893_b200 import verify as V
    from paper_2605_19893_b200.workload import chain_tree_mask

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = llama_cfg(a.layers)
    L, g, nq = a.layers, a.gamma, 1 + a.gamma
    mode = V.MODE_EXACT if a.mode == "exact" else V.MODE_APPROX
    roles, source = V.resolve_layer_roles(reuse_set(a.schedule, L), L)
    H, dh, Hq = cfg.n_kv_heads, cfg.d_head, cfg.n_q_heads
    shards = sharding.shard_plan(a.total_requests, world, rank, H)
    R = len(shards)
    heads = [s.kv_heads() for s in shards]
    units_this_rank = sum(s.fraction for s in shards) * nq  # query-tokens completed per step
    extra_rows = (a.warmup + a.steps + 4) * (a.accept + 1)  # e2e steps grow the context
    cap = a.ctx + extra_rows
    gen = torch.Generator(device=dev)

    def urand(*shape, dtype=torch.float32):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(dtype)

    pos = np.array([a.ctx - 1 + i for i in range(nq)], np.int64)
    tmask = chain_tree_mask(g)
    caches, batches, sets, outs, inbufs, pes = [], [], [], [], [], []
    for r in range(R):
        gen.manual_seed(sharding.request_seed(shards[r].request))
        # one packed row per layer -- q | gates | draft K | draft V -- so the
        # e2e path moves a layer's inputs with ONE host->device copy
        parts = [((nq, Hq, dh), torch.float32), ((nq, Hq, 3), torch.float32),
                 ((max(g, 1), H, dh), torch.bfloat16), ((max(g, 1), H, dh), torch.bfloat16)]
        sizes = [int(np.prod(sh)) * torch.tensor([], dtype=dt).element_size() for sh, dt in parts]
        offs = np.concatenate([[0], np.cumsum([(nb + 255) // 256 * 256 for nb in sizes])]).tolist()
        packed = torch.zeros(L, offs[-1], dtype=torch.uint8, device=dev)  # 256 B-aligned parts
        views = [packed[:, o:o + nb].view(dt).view(L, *sh)
                 for (sh, dt), nb, o in zip(parts, sizes, offs)]
        qa, ga, tka, tva = views
        qa.copy_(urand(L, nq, Hq, dh))
        ga.copy_(torch.rand(L, nq, Hq, 3, generator=gen, device=dev) * 0.6 + 0.2)
        tka.copy_(urand(L, max(g, 1), H, dh, dtype=torch.bfloat16))
        tva.copy_(urand(L, max(g, 1), H, dh, dtype=torch.bfloat16))
        inbufs.append(packed)
        pe = urand(cfg.l, dh) * 0.1
        pes.append(pe)
        cr, br, sr, orr = [], [], [], []
        for j in range(L):
            c = V.LayerCache(cfg, cap, device=dev)
            c.k[:a.ctx].copy_(urand(a.ctx, H, dh, dtype=torch.bfloat16))
            c.v[:a.ctx].copy_(urand(a.ctx, H, dh, dtype=torch.bfloat16))
            c.rows = a.ctx
            c.extend_compressed(pe)
            cr.append(c)
            br.append(V.DraftBatch(pos=pos.copy(), tree_mask=tmask, q=qa[j], gates=ga[j],
                                   tree_k=tka[j], tree_v=tva[j]))
            sr.append(V.IndexSets.empty(nq, cfg.n, dev))
            orr.append(torch.zeros(nq, Hq, dh, device=dev))
        caches.append(cr)
        batches.append(br)
        sets.append(sr)
        outs.append(orr)
    ws = V.Workspace(cfg, nq, cap, device=dev, batch=min(R, 16))  # C4: batched routing
    torch.cuda.synchronize()

    def layer(j, role=None):
        rj = int(roles[j]) if role is None else role
        # index sets: a refresh layer's own, a reuse layer's source layer's
        src = j if roles[j] == V.ROLE_REFRESH else int(source[j])
        if R == 1:
            V.nsa_verify(cfg, caches[0][j], batches[0][j], sets[0][src], outs[0][j], ws, a.group,
                         mode, rj, kv_heads=heads[0])
            return
        # C4: one batched call per layer over this GPU's requests
        V.nsa_verify_batched(cfg, [caches[r][j] for r in range(R)], [batches[r][j] for r in range(R)],
                             [sets[r][src] for r in range(R)], [outs[r][j] for r in range(R)], ws,
                             a.group, mode, [rj] * R, kv_heads=heads)

    def step():
        for j in range(L):
            layer(j)

    n_refresh = int((roles == V.ROLE_REFRESH).sum())
    att_launches_per_layer = (R + 7) // 8 if R > 1 else 1        # batched attend: 8 requests each
    route_launches_per_layer = (R + 15) // 16 if R > 1 else 1    # batched routing: 16 each
    launches_per_step = n_refresh * route_launches_per_layer + L * att_launches_per_layer

    def progress(msg):
        if os.environ.get("SPECSV_BENCH_PROGRESS"):
            print(f"[bench r{rank}] {msg}", file=sys.stderr, flush=True)

    def capture(fn):
        gph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(device=dev)
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(gph, stream=cs):
                fn()
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        return gph

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    progress("eager steps done")
    graph = None if a.no_graph else capture(step)
    progress("step graph captured")

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        run_step()
    barrier()
    progress("warmup done")
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(a.steps):
            run_step()
        ev1.record(stream)
        barrier()
    ms_rank = ev0.elapsed_time(ev1) / a.steps
    value, ms = sharding.job_throughput(units_this_rank, ms_rank, dev)
    progress("timed steps done")

    # ---- kernel-level roofline of the dominant kernel (the fused attend) and
    # the routing launches, each captured alone over all L layers (graphs on
    # the launching stream, CUDA events around the replay)
    def attend_all():
        for j in range(L):
            layer(j, V.ROLE_REUSE)  # reuse = the fused attend launch(es) only

    def route_refresh_all():
        for j in range(L):
            if roles[j] == V.ROLE_REFRESH:
                layer(j, V.ROLE_REFRESH)

    g_att = capture(attend_all)
    g_rf = capture(route_refresh_all)
    att_ms, rf_ms = [], []
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for rep in range(6):
        e[0].record(stream)
        g_att.replay()
        e[1].record(stream)
        g_rf.replay()
        e[2].record(stream)
        torch.cuda.synchronize()
        if rep > 0:
            att_ms.append(e[0].elapsed_time(e[1]) / (L * att_launches_per_layer))
            rf_ms.append(e[1].elapsed_time(e[2]) / max(1, n_refresh))
    attend_ms = float(np.median(att_ms))                      # per attend launch
    refresh_layer_ms = float(np.median(rf_ms))                # route + attend of a refresh layer
    route_ms = (refresh_layer_ms - attend_ms * att_launches_per_layer) / route_launches_per_layer
    progress("kernel timings done")

    # ---- algorithmic bytes from the actual index sets, summed over
    # this rank's requests; KV bytes per verified query vs the no-reuse
    # per-query decode of the same queries (the north star's counter)
    alg_att, alg_route, uniq, noreuse = [], [], [], []
    for j in range(L):
        src = j if roles[j] == V.ROLE_REFRESH else int(source[j])
        b_att = b_route = b_nr = 0
        for r in range(R):
            idx = sets[r][src].idx.cpu().numpy()
            cnt = sets[r][src].count.cpu().numpy()
            frac = shards[r].fraction
            ba = V.algorithmic_bytes(cfg, a.ctx, pos, V.ROLE_REUSE, idx, cnt, mode, a.group)
            bf = V.algorithmic_bytes(cfg, a.ctx, pos, V.ROLE_REFRESH, idx, cnt, mode, a.group)
            b_att += ba * frac
            b_route += bf - ba  # routing is replicated on head-group shards
            for q in range(nq):  # one single-query decode per query, its own set, refresh
                b_nr += frac * V.algorithmic_bytes(cfg, a.ctx, pos[q:q + 1], V.ROLE_REFRESH,
                                                   idx[q:q + 1], np.maximum(cnt[q:q + 1], 0),
                                                   V.MODE_EXACT, 1)
            if r == 0:
                uniq.append(len(set(idx[cnt > 0].ravel().tolist()) - {-1}))
        alg_att.append(b_att)
        alg_route.append(b_route)
        noreuse.append(b_nr)
    bytes_att_launch = float(np.mean(alg_att)) / att_launches_per_layer
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks
                else "B200_PROFILING.md fallback")
    achieved = bytes_att_launch / (attend_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(a.workload, min(R, 8) if R > 1 else 1)
    step_bytes = sum(alg_att) + sum(alg_route[j] for j in range(L) if roles[j] == V.ROLE_REFRESH)
    step_noreuse = sum(noreuse)
    q_done = units_this_rank  # query-tokens this rank completes per step
    kv_per_query = {"verify": step_bytes / q_done, "no_reuse_decode": step_noreuse / q_done,
                    "ratio": step_noreuse / max(step_bytes, 1.0),
                    "what": "algorithmic HBM bytes per verified query-token over one step (all "
                            "layers, routing included): this verify vs 1+gamma independent "
                            "single-query NSA decodes (own index sets, no cross-query reuse)"}

    # ---- per-query NSA decode on the same GPU and caches (north star: verify
    # >= 3x faster), request 0: the 1 + gamma queries as sequential
    # single-query decodes, every layer refreshing its own indices
    decode = None
    if not a.skip_decode_baseline:
        ws1 = V.Workspace(cfg, 1, cap, device=dev)
        pos1 = np.array([a.ctx - 1], np.int64)
        dq = []
        for j in range(L):
            for i in range(nq):
                b1 = V.DraftBatch(pos=pos1, tree_mask=chain_tree_mask(0), q=batches[0][j].q[i:i + 1],
                                  gates=batches[0][j].gates[i:i + 1], tree_k=None, tree_v=None)
                dq.append((j, b1, V.IndexSets.empty(1, cfg.n, dev), torch.zeros(1, Hq, dh, device=dev)))

        def decode_all():
            for j, b1, s1, o1 in dq:
                V.nsa_verify(cfg, caches[0][j], b1, s1, o1, ws1, 1, V.MODE_EXACT, V.ROLE_REFRESH,
                             kv_heads=heads[0])

        g_dec = capture(decode_all)
        dsteps = max(2, a.steps // 4)
        for _ in range(2):
            g_dec.replay()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(dsteps):
            g_dec.replay()
        ev1.record(stream)
        torch.cuda.synchronize()
        dms = ev0.elapsed_time(ev1) / dsteps
        dbytes = 0
        for j, b1, s1, o1 in dq:
            dbytes += shards[0].fraction * V.algorithmic_bytes(
                cfg, a.ctx, pos1, V.ROLE_REFRESH, s1.idx.cpu().numpy(),
                np.maximum(s1.count.cpu().numpy(), 0), V.MODE_EXACT, 1)
        dgbs = dbytes / (dms * 1e-3) / 1e9
        verify_ms_one_request = ms_rank / R
        decode = {"value": nq * shards[0].fraction / (dms * 1e-3), "unit": UNIT, "ms_per_step": dms,
                  "what": f"{nq} sequential single-query NSA decodes per layer (C=1, gamma=0, "
                          f"refresh every layer), {L} layers, request 0 of rank 0, same GPU and caches",
                  "verify_speedup": dms / verify_ms_one_request,
                  "roofline": {"achieved": dgbs, "peak": peak, "unit": "GB/s", "frac": dgbs / peak,
                               "alg_bytes_per_step": dbytes}}
        progress("decode baseline done")

    # ---- e2e through the public API on REAL steps: each step copies its inputs
    # from pinned host memory, re-issues every layer's verify call with this
    # step's positions and rows (eager: host work in the timed region), commits
    # `accept` draft rows + the next root into every layer (the context grows)
    # and reads the last layer's output back
    # every step verifies new draft queries: a ring of input sets (q, gates, draft
    # rows), each copied host->device by the step that uses it
    ring = 4
    hin_ring = []
    for k in range(ring):
        if k > 0:
            gen.manual_seed(sharding.request_seed(shards[0].request) + 7919 * k)
            for r in range(R):  # the same distributions as the first set
                for j in range(L):
                    b = batches[r][j]
                    b.q.copy_(urand(*b.q.shape))
                    b.gates.copy_(torch.rand(*b.gates.shape, generator=gen, device=dev) * 0.6 + 0.2)
                    b.tree_k.copy_(urand(*b.tree_k.shape, dtype=torch.bfloat16))
                    b.tree_v.copy_(urand(*b.tree_v.shape, dtype=torch.bfloat16))
        hin_ring.append([t.cpu().pin_memory() for t in inbufs])
    hin = hin_ring[0]
    step_no = [0]
    hout = [torch.empty(nq, Hq, dh, pin_memory=True) for _ in range(R)]
    h2d = sum(t.numel() * t.element_size() for t in hin_ring[0])
    d2h = sum(t.numel() * t.element_size() for t in hout)
    acc = max(0, min(a.accept, g))
    slots = list(range(acc)) + ([acc] if acc < g else [])  # accepted drafts, then the bonus root's row
    host_s = [0.0]
    n_calls = [0]
    # Two device input sets (parity b = step % 2): while step s verifies from
    # set b, step s+1's inputs are copied host->device into set 1-b on a copy
    # stream (every timed step still copies one step's inputs and reads one
    # output back; the first timed step's inputs were copied by the last
    # warm-up step, the last timed step copies inputs no step uses).
    inbufs2 = [t.clone() for t in inbufs]
    batches2 = []
    for r in range(R):
        views = [inbufs2[r][:, o:o + nb].view(dt).view(L, *sh)
                 for (sh, dt), nb, o in zip(parts, sizes, offs)]
        batches2.append([V.DraftBatch(pos=batches[r][j].pos, tree_mask=tmask, q=views[0][j],
                                      gates=views[1][j], tree_k=views[2][j], tree_v=views[3][j])
                         for j in range(L)])
    sets_in = [(inbufs, batches), (inbufs2, batches2)]
    # one prepared C-ABI call per layer and input set (ctypes arguments built
    # once; rows and positions refreshed per step)
    prepared = [[], []]
    for b, (_, bset) in enumerate(sets_in):
        for j in range(L):
            src = j if roles[j] == V.ROLE_REFRESH else int(source[j])
            prepared[b].append(V.PreparedVerify(
                cfg, [caches[r][j] for r in range(R)], [bset[r][j] for r in range(R)],
                [sets[r][src] for r in range(R)], [outs[r][j] for r in range(R)], ws, a.group, mode,
                int(roles[j]), kv_heads=heads if R > 1 else heads[0]))
    copy_stream = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]  # set b's inputs landed
    done = [torch.cuda.Event(), torch.cuda.Event()]   # set b's readers (verify + commit) finished
    out_ready = torch.cuda.Event()

    # one commit call over every request's layers (the entry point takes a list
    # of independent caches), per input set
    commits = [[TR.PreparedCommit(cfg, [caches[r][j] for r in range(R) for j in range(L)],
                                  [bset[r][j].tree_k for r in range(R) for j in range(L)],
                                  [bset[r][j].tree_v for r in range(R) for j in range(L)], slots,
                                  [pes[r] for r in range(R) for j in range(L)])]
               if slots else [] for _, bset in sets_in]
    host_parts = {"copies": 0.0, "verify_calls": 0.0, "readback": 0.0, "commit": 0.0}
    host_role = {int(V.ROLE_REFRESH): 0.0, int(V.ROLE_REUSE): 0.0}

    variant = os.environ.get("SPECSV_E2E_VARIANT", "")  # diagnostics only: drop one part of the step

    def copy_inputs(s_no, cur):
        """host->device copy of step s_no's inputs into set s_no % 2, on the copy
        stream, once that set's previous readers (step s_no - 2) are done"""
        b = s_no % 2
        hin = hin_ring[s_no % ring]
        copy_stream.wait_event(done[b])
        with torch.cuda.stream(copy_stream):
            if variant != "nocopy":
                for r in range(R):
                    sets_in[b][0][r].copy_(hin[r], non_blocking=True)
            ready[b].record(copy_stream)

    def e2e_step():
        tA = time.perf_counter()
        s_no = step_no[0]
        step_no[0] += 1
        b = s_no % 2
        cur = torch.cuda.current_stream()
        if s_no == 0:  # (the first warm-up step copies its own inputs)
            for k in (0, 1):
                done[k].record(cur)
            copy_inputs(0, cur)
        copy_inputs(s_no + 1, cur)  # the next step's inputs, under this step's kernels
        tB = time.perf_counter()
        cur.wait_event(ready[b])
        for j in range(L):
            t0 = time.perf_counter()
            prepared[b][j].run()
            dt = time.perf_counter() - t0
            host_s[0] += dt
            n_calls[0] += 1
            host_role[int(roles[j])] += dt
        tC = time.perf_counter()
        if variant != "nod2h":  # the step's result, read back on the copy stream
            out_ready.record(cur)
            copy_stream.wait_event(out_ready)
            with torch.cuda.stream(copy_stream):
                for r in range(R):
                    hout[r].copy_(outs[r][L - 1], non_blocking=True)
        tD = time.perf_counter()
        for pc in commits[b] if variant != "nocommit" else []:  # rows + positions advance
            pc.run(cur)
            for r in range(R):
                new_pos = np.array([caches[r][0].rows - 1 + i for i in range(nq)], np.int64)
                for j in range(L):
                    batches[r][j].pos = new_pos
                    batches2[r][j].pos = new_pos
        done[b].record(cur)
        tE = time.perf_counter()
        host_parts["copies"] += tB - tA
        host_parts["verify_calls"] += tC - tB
        host_parts["readback"] += tD - tC
        host_parts["commit"] += tE - tD

    for _ in range(max(3, a.warmup)):
        e2e_step()
    barrier()
    host_s[0], n_calls[0] = 0.0, 0
    for k in host_parts:
        host_parts[k] = 0.0
    for k in host_role:
        host_role[k] = 0.0
    t0w = time.perf_counter()
    ev0.record(stream)
    for _ in range(a.steps):
        e2e_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0w) * 1e3 / a.steps
    e2e_rank_ms = max(ev0.elapsed_time(ev1) / a.steps, wall_ms)
    e2e_value, e2e_ms = sharding.job_throughput(units_this_rank, e2e_rank_ms, dev)
    host_us = host_s[0] / max(1, n_calls[0]) * 1e6
    progress("e2e done")

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not a.skip_cpu_baseline:
        threads = a.cpu_threads or os.cpu_count() or 1
        ref = CpuReference(a, threads)
        rate, sample = ref.measure(a.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": ref.kind, "sample": sample,
               **ref.describe()}
    clocks = clk.summary()
    line = {
        "metric": metric_for(a.ctx, a.gamma), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (U[-1,1] KV and queries, random-init; no checkpoint)",
        "config": workload_config(a, world),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "advancing": True, "ms_per_step": e2e_ms,
                "host_us_per_call": host_us, "accepted_rows_per_step": len(slots),
                "host_us_per_step": {k: v / a.steps * 1e6 for k, v in host_parts.items()},
                "host_us_per_call_by_role": {
                    "refresh": host_role[int(V.ROLE_REFRESH)] / max(1, a.steps * n_refresh) * 1e6,
                    "reuse": host_role[int(V.ROLE_REUSE)] / max(1, a.steps * (L - n_refresh)) * 1e6},
                "what": "eager C-ABI calls per layer with each step's positions/rows, pinned "
                        "host->device inputs, accepted-row commit + compressed append, "
                        "last layer's output device->host"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": f"profiles/{traffic_src}" if traffic_src else None,
                     "frac_vs_spec_8000": achieved / 8000.0,
                     "kernel": ("nsa_attend_kernel" if R == 1 else "nsa_attend_batch_kernel")
                               + " (fused cmp+slc+win+gate, one launch per layer"
                               + ("" if R == 1 else ", up to 8 requests") + ")",
                     "alg_bytes_per_launch": bytes_att_launch, "launch_ms": attend_ms,
                     "peak_source": peak_src},
        "kv_bytes_per_query": kv_per_query,
        "cpu_baseline": cpu,
        "decode_baseline": decode,
        "clocks": clocks,
        "gpu_launches": launches_per_step * a.steps,
        "detail": {
            "per_layer_us_step_avg": ms * 1e3 / L,
            "attend_us_per_launch": attend_ms * 1e3, "route_us_per_launch": route_ms * 1e3,
            "route_alg_bytes_per_layer": float(np.mean(alg_route)),
            "step_alg_bytes_this_rank": step_bytes,
            "step_alg_GBps": step_bytes / (ms_rank * 1e-3) / 1e9,
            "step_frac_of_peak": step_bytes / (ms_rank * 1e-3) / 1e9 / peak,
            "unique_selected_blocks_per_layer": float(np.mean(uniq)),
            "refresh_layers": n_refresh, "reuse_layers": L - n_refresh,
            "route_exact_rescorings": ws.route_fallbacks(),
            "requests_this_rank": R, "graph": graph is not None,
            "shards_rank0": [(s.request, s.head_begin, s.head_count) for s in shards],
        },
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    a = parse(argv)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a, argv))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"[bench] note: --gpus {a.gpus} but WORLD_SIZE={world}; using {world}",
              file=sys.stderr)
    resolve_workload(a, world)
    if a.impl == "reference":
        run_reference_arm(a, world, rank)
    elif a.dry_run:
        run_dry(a, world, rank)
    else:
        run_ours(a, world, rank, local)


if __name__ == "__main__":
    main()
