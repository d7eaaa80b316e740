#!/usr/bin/env python
"""bench.py -- Andes scheduling decisions/s at 64K live requests on B200 (BASELINE config 3),
plus QoE-eval token-events/s against the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full Andes decision (S0-S6: trigger, timeline QoE scan, gains for every
B = 1..256, Algorithm 1 per B, best B, preemption cap) over the config-3 snapshot, captured
once in a CUDA graph and replayed; inputs resident in HBM; L2 flushed (256 MiB write)
between timed steps; device time from CUDA events.  Under torchrun (N > 1) every rank
schedules its own independent 64K-request instance (weak scaling, no data-path
collective); rank 0 prints the JSON line with the max-over-ranks time.

The line also carries config5_sweep (1024 independent scenarios split over the ranks, end-of-trace
QoE mean per scenario) and config4_sharded: the 2^20-request population (BASELINE config 4) split
into contiguous shards over the ranks, one decision through the multi-GPU entry point
(andes_schedule_shard; NCCL all-gathers between its steps at N > 1), device time max over ranks.

--impl reference times the CPU oracle (oracle/, plain C) on the same workload: one full
config-3 decision per step, its per-B walks on every host core (rank 0 only).

--gpus N without a launcher re-executes itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Andes sched decisions/s at 64K live requests; QoE-eval token-events/s vs HBM"
WORKLOAD = ("config3: burst arrivals at 2x capacity, 64K live requests (ShareGPT-shaped), 50/50 "
            "reading/listening, B=1..256 (pruning off), M=163840, dt=2s, preemption cap 16")
UNIT = "decisions/s"
KERNELS_PER_DECISION = 5  # k_prep, k_qoe_scan, k_state, k_compact, k_select


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _ncu_traffic():
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
    kernels from the committed `ncu --set full` captures (profiles/ncu_traffic.json), or {}."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


def _hbm_peak():
    p = _peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler during the timed region (recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def start(self, load=None, load_s=0.6):
        """Start sampling; wait for the first sample, then run `load` (the timed work itself,
        untimed) for load_s seconds so the samples see the clocks under this load."""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 5.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)
        if load is not None:
            t0 = time.time()
            while time.time() - t0 < load_s:
                load()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        if sm:
            out["sm_mhz"] = statistics.median(sm)
            out["sm_max_mhz"] = float(rows[0][2])
            out["samples"] = len(sm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].strip() == "Active" and nm not in out["reasons"]:
                        out["reasons"].append(nm)
        return out


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        # test hooks for the N > 1 code path on a one-GPU box: every rank on cuda:0, gloo instead
        # of NCCL (NCCL refuses two ranks on one GPU); the driver's runs use neither
        if os.environ.get("ANDES_BENCH_ONE_GPU") == "1":
            lr = 0
        torch.cuda.set_device(lr)
        dist.init_process_group(os.environ.get("ANDES_DIST_BACKEND", "nccl"))
        return dist, dist.get_rank(), ws, lr
    return None, 0, 1, 0


def _max_over_ranks(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _token_events(snap):
    import numpy as np
    t = snap.now_us + snap.horizon_us - snap.arrival_us
    m = np.where(t < snap.ttft_us, 0, (t - snap.ttft_us.astype(np.int64)) // snap.period_us + 1)
    m = np.minimum(m, snap.max_total)
    return int(np.minimum(snap.n_deliv, m).sum())


def _tile(snap, reps):
    """reps copies of a snapshot (same shape/statistics), for the QoE-eval throughput run."""
    import workloads as W
    return W.tile(snap, reps)


def sweep_run(args, dist, rank, ws, lr, stream):
    """Config 5: 1024 independent scenarios (32 trace seeds x 32 load factors) split over the
    ranks (contiguous blocks, replicas only: no data-path collective), FINAL-mode QoE of every
    request and the mean per scenario (andes_qoe_scenario_mean); the means are gathered to rank 0
    at the end (the one exchange).  Inputs are larger than L2 (~4 GB of timestamps)."""
    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    import workloads as W

    dev = torch.device("cuda", lr)
    scen = W.config5_scenarios()
    S = len(scen)
    lo, hi = rank * S // ws, (rank + 1) * S // ws
    t0 = time.time()
    snap, off = W.sweep(scen[lo:hi])
    gen_s = time.time() - t0
    ctx = A.Context(max_requests=max(snap.n, 1), max_B=8, max_tokens=snap.n_tokens + 64, device=lr)
    req = A.requests_to(snap, device=dev)
    offd = torch.from_numpy(off.view(np.int32)).to(dev)
    with torch.cuda.stream(stream):
        for _ in range(2):
            ctx.qoe_scenario_mean(req, snap.n, offd, stream=stream)
        stream.synchronize()
        reps = max(3, min(args.steps, 10))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        if dist is not None:
            dist.barrier()
        a.record(stream)
        for _ in range(reps):
            mean, cnt = ctx.qoe_scenario_mean(req, snap.n, offd, stream=stream)
        b.record(stream)
        b.synchronize()
    ms = _max_over_ranks(dist, a.elapsed_time(b) / reps)
    tokens = int(_sum_over_ranks(dist, snap.n_tokens))
    nreq = int(_sum_over_ranks(dist, snap.n))
    if dist is not None:  # C4: the scenario means to every rank (rank 0 reports)
        allm = [torch.empty_like(mean) for _ in range(ws)]
        dist.all_gather(allm, mean.contiguous())
        mean = torch.cat(allm)
    mq = mean.cpu().numpy()
    rh = np.array([r for _, r in scen])
    by_rho = {f"{r:.2f}": float(mq[rh == r].mean()) for r in (0.5, 1.0, 1.5, 2.0)}
    bytes_ = 4 * tokens + 44 * nreq
    res = {"workload": "config5: 1024 scenarios (32 seeds x rho 0.50..2.05), ~2000*rho requests each, complete "
                       "ShareGPT-shaped timelines from the parametric load model; FINAL-mode QoE, mean per scenario",
           "scenarios": S, "requests": nreq, "token_events": tokens, "ms_per_sweep": ms,
           "scenarios_per_s": S / (ms / 1e3), "token_events_per_s": tokens / (ms / 1e3),
           "achieved_GBs": bytes_ / (ms / 1e3) / 1e9, "host_generation_s": round(gen_s, 1),
           "mean_qoe_at_rho": by_rho, "l2": "inputs ~4 GB > L2 (no flush needed)"}
    del ctx, req
    return res


def _sum_over_ranks(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def sharded_decision(args, dist, rank, ws, lr, stream, flush):
    """Config 4: 2^20 live requests sharded over the ws ranks (contiguous ranges), one full
    decision through andes_schedule_shard: five step graphs, the four all-gathers between them
    (NCCL over NVLink at ws > 1; a device copy at ws = 1).  Device time per decision, max over
    ranks, L2 flushed before each decision."""
    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    import workloads as W

    dev = torch.device("cuda", lr)
    big = W.config4()
    cuts = np.linspace(0, big.n, ws + 1).astype(np.int64)
    mine = W.shard(big, int(cuts[rank]), int(cuts[rank + 1]))
    ctx = A.Context(max_requests=max(mine.n, 1), max_B=256, max_tokens=mine.n_tokens + 64, device=lr)
    req = A.requests_to(mine, device=dev)
    tau = torch.from_numpy(big.tau_us.view(np.int32)).to(dev)
    sh = ctx.shard_init(ws, rank, 256)
    send, recv = ctx.alloc_shard_buffers(sh)
    out = ctx.alloc_shard_decision(mine.n, 256)
    ag = A.torch_allgather() if dist is not None else (lambda a, b: b.copy_(a))
    kw = dict(preempt_cap=big.preempt_cap, flags=A.ANDES_FORCE, stream=stream)

    def step(s_):
        ctx.schedule_shard(sh, s_, req, mine.n, big.now_us, big.horizon_us, tau, big.kv_capacity, out,
                           recv=recv[s_ - 1] if s_ else None, send=send[s_] if s_ < A.SHARD_ROUNDS else None, **kw)

    def eager():
        for s_ in range(A.SHARD_STEPS):
            step(s_)
            if s_ < A.SHARD_ROUNDS:
                ag(send[s_], recv[s_])

    def timed(ag_fn, tag):
        """Capture the decision (five steps + four all-gathers with ag_fn) in one graph (per-step
        graphs with eager all-gathers if the collective cannot be captured), replay, time."""
        nonlocal ag
        ag = ag_fn
        with torch.cuda.stream(stream):
            for _ in range(3):
                eager()
            stream.synchronize()
            launch = f"one CUDA graph: 5 steps + 4 all-gathers ({tag})"
            try:
                g1 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g1, stream=stream):
                    eager()
                g1.replay()
                stream.synchronize()

                def decide():
                    g1.replay()
            except Exception as ex:  # noqa: BLE001 -- reported in the line
                launch = f"5 step CUDA graphs + 4 eager all-gathers ({tag}; capture failed: {type(ex).__name__})"
                stream.synchronize()
                graphs = []
                for s_ in range(A.SHARD_STEPS):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        step(s_)
                    graphs.append(g)

                def decide():
                    for s_ in range(A.SHARD_STEPS):
                        graphs[s_].replay()
                        if s_ < A.SHARD_ROUNDS:
                            ag(send[s_], recv[s_])

            for _ in range(max(args.warmup, 3)):
                flush.zero_()
                decide()
            stream.synchronize()
            ms = []
            for _ in range(args.steps):
                flush.zero_()
                if dist is not None:
                    dist.barrier()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                decide()
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
        return ms, launch

    ms, launch = timed(ag, "NCCL at world > 1, a device copy at world 1")
    collectives = {}
    if dist is not None:
        # the same decision with the exchanges as device collectives over peer memory (andes_comm:
        # CUDA IPC mappings of each rank's arena, P2P stores over NVLink; no NCCL)
        collectives[f"{dist.get_backend()}_ms_per_decision"] = _max_over_ranks(dist, sum(ms)) / args.steps
        try:
            comm, ok = None, 1
            try:
                comm = A.Comm(ws, rank, max(int(x) for x in sh.xbytes), device=lr)
                hs = [None] * ws
                dist.all_gather_object(hs, comm.handle)
                comm.connect(hs)
            except Exception:  # noqa: BLE001 -- every rank must agree before any waits on a peer
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                raise RuntimeError("andes_comm setup failed on some rank (CUDA IPC / peer access)")
            ms_c, launch_c = timed(comm.allgather, "andes_comm peer-memory all-gathers")
            collectives["peer_memory_ms_per_decision"] = _max_over_ranks(dist, sum(ms_c)) / args.steps
            collectives["peer_memory_launch"] = launch_c
        except Exception as ex:  # noqa: BLE001 -- reported in the line
            collectives["peer_memory_error"] = f"{type(ex).__name__}: {ex}"[:200]
    total = _max_over_ranks(dist, sum(ms))
    sc = out.scalars.cpu().numpy().view(np.uint32).copy()
    res = {"workload": "config4: 2^20 live requests (config 3 x16, running batch in the first copy), "
                       "contiguous shards over the ranks, B=1..256, M=163840, preemption cap 16",
           "n_requests": int(big.n), "world": ws, "requests_per_rank": int(mine.n),
           "ms_per_decision": total / args.steps, "decisions_per_s": args.steps / (total / 1e3),
           "launch": launch,
           "collectives": collectives or None,
           "xbytes_per_round": [int(x) for x in sh.xbytes],
           "decision": {k: int(v) for k, v in zip(A.SC_NAMES, sc)}}
    if dist is not None:
        t = torch.from_numpy(sc.view(np.int32)).to(dev)
        allsc = [torch.empty_like(t) for _ in range(ws)]
        dist.all_gather(allsc, t)
        res["replicated_scalars_identical"] = all(bool(torch.equal(x, t)) for x in allsc)
    else:
        # world 1: the sharded decision must equal andes_schedule on the same population
        ref = ctx.schedule(req, mine.n, big.now_us, big.horizon_us, tau, big.kv_capacity,
                           preempt_cap=big.preempt_cap, flags=A.ANDES_FORCE)
        torch.cuda.synchronize()
        res["equals_single_gpu_decision"] = bool(
            np.array_equal(ref.scalars.cpu().numpy(), out.scalars.cpu().numpy())
            and np.array_equal(ref.V.cpu().numpy(), out.V.cpu().numpy())
            and np.array_equal(ref.serve_mask.cpu().numpy()[:mine.n], out.serve_mask.cpu().numpy()[:mine.n]))
    del ctx, req
    return res


def _host_info():
    """Host cores this process may use and the CPU model (lscpu), for the oracle baselines."""
    import oracle
    model = ""
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return oracle.nproc(), model


def _oracle_decision(oracle, snap, threads):
    return oracle.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                           preempt_cap=snap.preempt_cap, threads=threads)


def decision_trace(ctx, req, n, snap, tau, out, stream):
    """Stage breakdown of one decision from the kernels' own %globaltimer stamps (one store per
    CTA start and end by thread 0: the graph's launches and overlaps are not perturbed the way
    event records between kernels perturb them).  Internal hooks andes_debug_trace/_read."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    L = A.lib()
    L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
    L.andes_debug_trace.argtypes = [C.c_void_p, C.c_int]
    L.andes_debug_trace(ctx._h, 1)
    with torch.cuda.stream(stream):
        for _ in range(3):
            ctx.schedule(req, n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=stream,
                         preempt_cap=snap.preempt_cap, flags=A.ANDES_FORCE)
        stream.synchronize()
        L.andes_debug_trace(ctx._h, 0)
        L.andes_debug_trace(ctx._h, 1)  # fresh stamps
        # the decision captured into a CUDA graph and replayed, as the timed steps run it; every
        # replay overwrites the stamps (later times), so they describe the last replay
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            ctx.schedule(req, n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=stream,
                         preempt_cap=snap.preempt_cap, flags=A.ANDES_FORCE)
        for _ in range(3):
            g.replay()
        stream.synchronize()
        del g
    tr = np.zeros(1 << 16, np.uint64)
    L.andes_debug_read(ctx._h, 7, tr.ctypes.data, tr.nbytes)
    L.andes_debug_trace(ctx._h, 0)
    tr = tr.astype(np.int64)

    def span(lo, hi):
        x = tr[lo:hi].reshape(-1, 2)
        return x[x[:, 0] > 0]
    pr, sc, st, cp, sel = span(7000, 8024), span(5000, 7000), span(3000, 4024), span(8100, 9124), span(0, 512)
    if not (len(pr) and len(sc) and len(cp) and len(sel)):
        return None
    t0 = pr[:, 0].min()
    us = lambda v: round((int(v) - t0) / 1e3, 2)  # noqa: E731
    fin = [us(tr[k]) for k in (2100, 2105) if tr[k]]
    stages = {"prep": [0.0, us(pr[:, 1].max())], "scan": [us(sc[:, 0].min()), us(sc[:, 1].max())]}
    if len(st):  # k_state (absent when the state is fused into the scan)
        stages["state"] = [us(st[:, 0].min()), us(st[:, 1].max())]
    stages.update({"compact": [us(cp[:, 0].min()), us(cp[:, 1].max())],
                   "select": [us(sel[:, 0].min()), us(sel[:, 1].max())], "finalize": fin})
    names = list(stages)[:-1]
    gaps = {f"{a}->{b}": round(stages[b][0] - stages[a][1], 2) for a, b in zip(names, names[1:])}
    return {"source": "in-kernel %globaltimer stamps (CTA start/end), one config-3 decision replayed from a CUDA graph as in the timed steps (the last of three replays), L2 warm",
            "stages_us_from_prep_start": stages, "gaps_us": gaps}


def serving_sim(args, lr, stream):
    """NEXT-3: the serving loop on the device (andes_simulate) over cyclic-burst traces at four
    load factors, Andes' priority (gain / l, Eq. 6) vs LQSF (raw gain, reading R21), zero
    preemption overhead; end-of-trace average QoE (FINAL mode, mean over requests with tokens,
    P:L719) per load -- the fig:e2e-intensity analog without models (iteration latency = the
    synthetic tau(B) table).  Wall time of the whole loop (one host read per iteration)."""
    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    import workloads as W

    dev = torch.device("cuda", lr)
    tau = torch.from_numpy(W.tau_table().view(np.int32)).to(dev)
    rhos = (0.5, 1.0, 1.5, 2.0)
    seeds = (1,)
    res = {"andes": {}, "lqsf": {}}
    iters = 0
    t_all = 0.0
    traces = [(sd, rho, W.sim_trace(sd, rho, window_s=60.0, rate_at_rho1=8.0)) for rho in rhos for sd in seeds]
    nmax = max(t["n"] for _, _, t in traces)
    tmax = max(t["tl_len"] for _, _, t in traces)
    ctx = A.Context(max_requests=nmax, max_B=256, max_tokens=tmax + 64, device=lr)
    for pol, fl in (("andes", 0), ("lqsf", A.ANDES_LQSF)):
        for sd, rho, tr in traces:
            t0 = time.perf_counter()
            g, pool, t, st = ctx.simulate(tr, tau, W.KV_CAPACITY, flags=fl, stream=stream)
            stream.synchronize()
            t_all += time.perf_counter() - t0
            iters += st["iterations"]
            n = tr["n"]
            req = {"arrival_us": t["arrival_us"], "ttft_us": t["ttft_us"], "period_us": t["period_us"],
                   "ctx_len": t["prompt_len"], "n_deliv": g, "max_total": torch.full((n,), -1, dtype=torch.int32, device=dev),
                   "start_off_us": None, "rank": torch.arange(n, dtype=torch.int32, device=dev),
                   "running": torch.zeros(n, dtype=torch.uint8, device=dev), "tl_base": t["tl_base"], "tl_pool": pool}
            q, q64, sd_, sw_, m = ctx.qoe_eval(req, n, 0, A.ANDES_EVAL_FINAL, stream=stream)
            qq = q64.cpu().numpy()[g.cpu().numpy() > 0]
            res[pol].setdefault(f"{rho:.2f}", []).append(float(qq.mean()) if qq.size else 0.0)
    out = {"workload": ("NEXT-3 serving loop on the device: cyclic-burst traces (60 s, intensity 2, 35% burst), "
                        "rho 0.5..2.0 x 8 req/s, ShareGPT-shaped, 50/50 reading/listening, "
                        "M=163840, B=1..256, tau(B)=20ms+0.8ms*B, zero preemption overhead"),
           "avg_qoe_by_rho": {pol: {k: round(float(np.mean(v)), 4) for k, v in d.items()} for pol, d in res.items()},
           "decisions": iters, "wall_s": round(t_all, 2), "decisions_per_s": iters / t_all if t_all else None}
    del ctx
    return out


def e2e_incremental(args, dist, snap, ws, lr, stream):
    """The serving loop through the public API with a device-resident Request Tracker.  One
    serving iteration -- (a) the copy of the decision time and of the previous iteration's
    delivered tokens (request index, delivery time) from pinned host memory, (b) their in-place
    append (andes_tracker_append_dev: count read on the device; the decision's serve mask becomes
    the running set), (c) the full config-3 decision (andes_schedule with now_dev: time read on the
    device), (d) the read-back of the decision to pinned host memory (scalars, V, admit and
    preempt lists) -- is captured ONCE into a CUDA graph; every step the host writes the new time
    and deltas into the pinned staging buffers, replays the graph, synchronises and updates the
    served set from the admit / preempt lists.  Wall time per step; the population evolves as in
    serving (the clock advances by tau(B*) per step)."""
    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    import workloads as W

    dev = torch.device("cuda", lr)
    steps = max(5, min(args.steps, 40))
    sn = W.with_room(snap, steps + 8)
    n = sn.n
    ctx = A.Context(max_requests=n, max_B=256, max_tokens=sn.n_tokens + 64, device=lr)
    req = A.requests_to(sn, device=dev)
    tau = torch.from_numpy(sn.tau_us.view(np.int32)).to(dev)
    out = ctx.alloc_decision(n, 256)
    maxc = min(n, 1024)  # deltas per iteration: one token per served request (the batch, <= 1024)
    pmax = min(n, 4096)  # preempt list bound: the running set (<= 4096)
    # zero-copy in both directions (pinned host memory is device-mapped under UVA): the decision's
    # last kernel writes its head (scalars, V, admit, the first pmax preempt slots) and the next
    # batch as an index list into a pinned export block; the engine (here: the host loop) runs that
    # batch and reports one delivery time per served request into pinned memory; the next
    # iteration's tracker update reads the batch list, its count (the realized scalar) and the times
    # from there, and the decision its time -- no copy nodes in the iteration's graph
    hnow = torch.zeros(1, dtype=torch.int64).pin_memory()
    hts = torch.zeros(maxc, dtype=torch.int64).pin_memory()
    ebytes = A.decision_export_bytes(256, pmax, maxc)
    hexp = torch.zeros(ebytes, dtype=torch.uint8).pin_memory()
    np_sc, _, np_adm, np_pre, np_srv = A.decision_export_views(hexp, 256, pmax, maxc)
    o_srv = 32 + 12 * 256 + 4 * pmax
    srv_t = hexp[o_srv:o_srv + 4 * maxc].view(torch.int32)  # the exported batch (tracker idx)
    np_done = A.decision_export_done(hexp, 256, pmax, maxc)  # polled instead of a stream sync
    cnt_t = hexp[4:8].view(torch.int32)  # scalars[ANDES_SC_REALIZED] (tracker count)
    np_now, np_ts = hnow.numpy(), hts.numpy()
    h2d = d2h = 0  # bytes the kernels read / write over PCIe per step (the used slots)
    kw = dict(preempt_cap=sn.preempt_cap, flags=A.ANDES_FORCE, stream=stream, export_host=hexp, export_preempt=pmax,
              export_served=maxc)

    def iteration():
        ctx.tracker_append_dev(req, n, srv_t, hts, cnt_t, serve_mask=out.serve_mask, stream=stream)
        ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=hnow, **kw)

    now = sn.now_us
    with torch.cuda.stream(stream):
        # iteration 0 (eager): the first decision on the snapshot as it is; no deliveries yet
        ctx.schedule(req, n, now, sn.horizon_us, tau, sn.kv_capacity, out=out, **kw)
        stream.synchronize()
        graph = None
        times = []
        for k in range(steps + 3):
            t0 = time.perf_counter()
            # the engine runs the exported batch: one token per request at now + tau(B*)
            cnt = int(np_sc[1])
            now += int(sn.tau_us[max(int(np_sc[0]), 1) - 1])
            assert cnt <= maxc and int(np_sc[3]) <= pmax
            np_now[0] = now
            np_ts[:cnt] = now
            np_done[0] = 0
            if graph is None:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    iteration()
            graph.replay()
            t_spin = time.perf_counter()
            while np_done[0] == 0:  # the export's completion word (written last, system fence)
                if time.perf_counter() - t_spin > 10.0:
                    stream.synchronize()
                    raise RuntimeError("e2e: the decision export never completed")
            dt = time.perf_counter() - t0
            if k >= 3:
                times.append(dt)
                h2d += 8 + 4 + 12 * cnt  # time, count, batch list and delivery times read by the kernels
                d2h += 32 + 8 * 256 + 4 * (int(np_sc[2]) + min(int(np_sc[3]), pmax) + int(np_sc[1]))
    tot = _max_over_ranks(dist, sum(times))
    del graph, ctx, req
    return {"value": ws * len(times) / tot, "unit": UNIT, "h2d_bytes_per_step": int(h2d // len(times)),
            "d2h_bytes_per_step": int(d2h // len(times)),
            "api": ("one CUDA graph per serving iteration, captured once and replayed: andes_tracker_append_dev "
                    "reading the previous iteration's deliveries (the exported batch list and its count, the "
                    "delivery times the host wrote) from pinned host memory, andes_schedule reading the decision "
                    "time from pinned memory (now_dev) and writing its head (scalars, V, admit list, preempt "
                    "list, the next batch) zero-copy into pinned memory (export_host); host: delivery times, "
                    "replay, poll the export's completion word; wall time per step; the config-3 population "
                    "evolves over the steps"),
            "steps": len(times), "ms_per_step": 1e3 * tot / len(times),
            "step_ms_min_median_max": [1e3 * min(times), 1e3 * sorted(times)[len(times) // 2], 1e3 * max(times)]}


def cpu_baseline(snap):
    """The oracle as it stands (plain C; its per-B walks split over every host core, SURVEY 8(d)
    "Oracle timing"), measured, nothing extrapolated: (i) one full threaded config-3 decision (the
    line's value); (ii) single-thread latency of a full config-1 and config-2 decision and of the
    config-3 decision restricted to B = 1..8 (labelled); (iii) QoE evaluation (S1 alone) over the
    2^20-request config-4 population on every core, in token-events/s.  About 15-25 s of CPU."""
    import oracle
    import workloads as W
    oracle.build()
    nproc, model = _host_info()
    t0 = time.perf_counter()
    _oracle_decision(oracle, snap, nproc)
    full_s = time.perf_counter() - t0
    lat = {}
    for name, sn in (("config1_8req", W.config1()), ("config2_4k", W.config2())):
        t0 = time.perf_counter()
        _oracle_decision(oracle, sn, 1)
        lat[name] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us[:8], snap.kv_capacity,
                    preempt_cap=snap.preempt_cap, B_cap=8)
    lat["config3_64k_B1to8_only"] = time.perf_counter() - t0
    big = W.tile(snap, 16)
    ev = _token_events(big)
    t0 = time.perf_counter()
    oracle.qoe_eval(big, big.now_us + big.horizon_us, threads=nproc)
    q_s = time.perf_counter() - t0
    return {"value": 1.0 / full_s, "unit": UNIT, "cores": nproc, "cpu_model": model, "kind": "oracle",
            "sample": (f"one full config-3 decision (64K requests, B=1..256, cap 16; oracle_schedule with its per-B "
                       f"walks on {nproc} threads): {full_s:.2f} s; measured, not extrapolated"),
            "single_thread_latency_s": {k: round(v, 4) for k, v in lat.items()},
            "qoe_eval": {"token_events_per_s": ev / q_s, "token_events": ev, "seconds": round(q_s, 3),
                         "threads": nproc, "workload": "S1 at now + dt over the 2^20-request config-4 population"}}


def run_reference(args):
    """--impl reference: the oracle (plain C CPU implementation of the paper's decision,
    oracle/) timed as it stands on this host's cores, one FULL config-3 decision per step (its
    independent per-B walks on every core; outputs identical for any thread count).  Rank 0
    only; other ranks exit without work."""
    dist_rank = int(os.environ.get("RANK", "0"))
    if dist_rank != 0:
        return
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    import workloads as W
    import oracle
    oracle.build()
    nproc, model = _host_info()
    snap = W.config3()
    # one full decision per step (~8 s on 16 cores): the warm-up is one decision and the timed
    # steps are capped so that the run ends within a few minutes (the line reports the steps it
    # ran; nothing is extrapolated)
    warm = min(args.warmup, 1)
    tw = time.perf_counter()
    for _ in range(max(warm, 1)):
        _oracle_decision(oracle, snap, nproc)
    t_one = time.perf_counter() - tw
    steps = max(1, min(args.steps, int(150.0 // max(t_one, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(steps):
        d = _oracle_decision(oracle, snap, nproc)
    total = time.perf_counter() - t0
    dt = total / steps
    v = 1.0 / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": steps,
            "requested_steps": args.steps, "requested_warmup": args.warmup,
            "warmup": max(warm, 1), "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic (workloads.config3, seed 1)",
            "config": {"workload": WORKLOAD},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nproc, "cpu_model": model, "kind": "oracle",
                             "sample": (f"each step: one full config-3 decision (64K requests, B=1..256, cap 16) by "
                                        f"oracle_schedule, per-B walks on {nproc} threads; {dt:.2f} s per decision, "
                                        f"{steps} decisions timed (B*={d.B_star}; steps capped to ~150 s)")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch

    import paper_2404_16283_b200 as A
    import workloads as W
    from paper_2404_16283_b200 import build as Bd

    dist, rank, ws, lr = _dist()
    Bd.build()
    dev = torch.device("cuda", lr)
    torch.cuda.set_device(dev)
    snap = W.config3(seed=1 + rank)
    n = snap.n
    ev_tokens = _token_events(snap)
    ctx = A.Context(max_requests=n, max_B=256, max_tokens=snap.n_tokens + 64, device=lr)
    req = A.requests_to(snap, device=dev)
    tau = torch.from_numpy(snap.tau_us.view(np.int32)).to(dev)
    stream = torch.cuda.Stream(device=dev)
    out = ctx.alloc_decision(n, 256)
    kw = dict(preempt_cap=snap.preempt_cap, flags=A.ANDES_FORCE)

    def decide(s):
        ctx.schedule(req, n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=s, **kw)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            decide(stream)
        stream.synchronize()
        # the timed graph carries no profiling events; a second, profiled graph (event records
        # between the kernels) gives the per-stage breakdown
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            decide(stream)
        ctx.profile_enable(True)
        pgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(pgraph, stream=stream):
            decide(stream)
        ctx.profile_enable(False)
        graph.replay()
        stream.synchronize()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(max(args.warmup, 3)):
            flush.zero_()
            graph.replay()
        stream.synchronize()

        # ---- per-stage breakdown (profiled graph, L2 flushed before each decision)
        stage_sum = [0.0] * A.N_STAGES
        for k in range(args.steps):
            flush.zero_()
            pgraph.replay()
            stream.synchronize()
            st = ctx.profile_read()
            stage_sum = [a + b for a, b in zip(stage_sum, st)]

        # ---- timed region: K decisions, L2 flushed between steps, CUDA events per step
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        clk = Clocks(lr)

        def _load():
            for _ in range(20):
                graph.replay()
            stream.synchronize()

        clk.start(load=_load)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            graph.replay()
            ends[k].record(stream)
            ends[k].synchronize()  # the next flush then covers the host's enqueue latency
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        clocks = clk.stop()
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total_ms = _max_over_ranks(dist, sum(step_ms))
        # L2-warm back-to-back replays (context)
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        w1.record(stream)
        w1.synchronize()
        warm_ms = w0.elapsed_time(w1) / args.steps

    sc = out.scalars.cpu().numpy().view(np.uint32)
    stage_ms = [x / args.steps for x in stage_sum]
    try:
        trace = decision_trace(ctx, req, n, snap, tau, out, stream)
    except Exception as ex:  # noqa: BLE001 -- the breakdown is context, the line must still print
        trace = {"error": f"{type(ex).__name__}: {ex}"}
    ms_per_step = total_ms / args.steps
    value = ws * args.steps / (total_ms / 1e3)

    # ---- roofline: the timeline scan (S1) is the path's one bandwidth-bound kernel; S3-S6
    # (k_state, k_compact, k_select) are latency-bound stages (one CTA per B)
    hbm_peak, hbm_src = _hbm_peak()
    names = A.STAGES
    dom = max(range(len(stage_ms)), key=lambda i: stage_ms[i])
    scan_i = names.index("scan")
    scan_bytes = 4 * snap.n_tokens + 44 * n  # one read of every timestamp + per-request SoA/state
    ach = scan_bytes / (stage_ms[scan_i] / 1e3) / 1e9
    roof = {"kernel": "k_qoe_scan (S1)", "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
            "frac": ach / hbm_peak, "traffic": _ncu_traffic().get("k_qoe_scan_config3"),
            "traffic_source": _ncu_traffic().get("source"), "peak_source": hbm_src,
            "algorithmic_bytes_per_launch": scan_bytes, "dominant_stage": names[dom],
            "note": ("S3-S6 (state, compact, select: candidate keys, Algorithm 1 per B, cap) are "
                     "latency-bound one-CTA-per-B stages without a throughput roofline; the scan is the "
                     "HBM-bound kernel. At 64K requests (38 MB) its launch is latency-bound (ramp-up and "
                     "tail of ~2.4 tiles per warp); its throughput roofline is qoe_eval.roofline (2^20 "
                     "requests, the same kernel)")}
    roof["stage_ms_event_graph"] = dict(zip(names, stage_ms))
    roof["stage_trace"] = trace
    roof["ib_evaluations_per_s"] = n * 256 / (ms_per_step / 1e3)
    try:  # issue-slot utilisation of every decision kernel, from the committed ncu capture
        roof["issue_active_pct_ncu"] = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                                   "profiles", "ncu_issue.json")))
    except (OSError, ValueError):
        roof["issue_active_pct_ncu"] = None
    roof["stage_share_event_graph"] = {k: v / sum(stage_ms) for k, v in zip(names, stage_ms)}

    # ---- S1 alone at scale: QoE-eval token-events/s on a 1M-request population (config-4 size)
    big = _tile(snap, 16)
    qctx = A.Context(max_requests=big.n, max_B=8, max_tokens=big.n_tokens + 64, device=lr)
    breq = A.requests_to(big, device=dev)
    big_events = _token_events(big)
    qctx.profile_enable(True)
    q_ms = []
    with torch.cuda.stream(stream):
        for k in range(max(args.warmup, 3) + 10):
            flush.zero_()
            qctx.qoe_eval(breq, big.n, big.now_us + big.horizon_us, A.ANDES_EVAL_INFLIGHT, stream=stream)
            st = qctx.profile_read()
            if k >= max(args.warmup, 3):
                q_ms.append(st)
    scan_ms = statistics.median([s[1] for s in q_ms])
    stage_sum_ms = statistics.median([s[0] + s[1] + s[2] for s in q_ms])
    # the whole call as a user makes it: no profiling events between its kernels
    qctx.profile_enable(False)
    c_ms = []
    with torch.cuda.stream(stream):
        for k in range(max(args.warmup, 3) + 10):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            qctx.qoe_eval(breq, big.n, big.now_us + big.horizon_us, A.ANDES_EVAL_INFLIGHT, stream=stream)
            b.record(stream)
            b.synchronize()
            if k >= max(args.warmup, 3):
                c_ms.append(a.elapsed_time(b))
    # the same call asking for the QoE only (AndesQoeOut.q; the other outputs NULL), and the
    # FINAL-mode evaluation (whole timelines, no clamp: the config-5 sweep's mode)
    def _whole_call(mode, outputs):
        ms = []
        with torch.cuda.stream(stream):
            for k in range(max(args.warmup, 3) + 10):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                qctx.qoe_eval(breq, big.n, big.now_us + big.horizon_us, mode, stream=stream, outputs=outputs)
                b.record(stream)
                b.synchronize()
                if k >= max(args.warmup, 3):
                    ms.append(a.elapsed_time(b))
        return statistics.median(ms)
    q_only_ms = _whole_call(A.ANDES_EVAL_INFLIGHT, ("q",))
    final_ms = _whole_call(A.ANDES_EVAL_FINAL, None)
    qctx.profile_enable(True)
    qoe_ms = statistics.median(c_ms)
    qbytes = 4 * big.n_tokens + 44 * big.n
    q_ach = qbytes / (scan_ms / 1e3) / 1e9
    qoe_eval = {"metric": "QoE-eval token-events/s", "value": big_events / (qoe_ms / 1e3),
                "unit": "token-events/s", "n_requests": big.n, "token_events": big_events,
                "pool_tokens": big.n_tokens, "ms_per_eval": qoe_ms, "scan_ms": scan_ms,
                "stage_sum_ms_profiled": stage_sum_ms,
                "whole_call_frac": qbytes / (qoe_ms / 1e3) / 1e9 / hbm_peak,
                "whole_call_q_only": {"ms_per_eval": q_only_ms, "frac": qbytes / (q_only_ms / 1e3) / 1e9 / hbm_peak,
                                      "note": "the same call with only AndesQoeOut.q requested (q64, S_delay, "
                                              "S_whole, m NULL)"},
                "whole_call_final_mode": {"ms_per_eval": final_ms,
                                          "frac": qbytes / (final_ms / 1e3) / 1e9 / hbm_peak,
                                          "note": "ANDES_EVAL_FINAL (every delivered token, no clamp), all outputs"},
                "roofline": {"kernel": "k_qoe_scan", "bound": "hbm", "achieved": q_ach, "peak": hbm_peak,
                             "unit": "GB/s", "frac": q_ach / hbm_peak,
                             "traffic": _ncu_traffic().get("k_qoe_scan_2p20"),
                             "algorithmic_bytes_per_launch": qbytes, "peak_source": hbm_src}}
    # the same population with unaligned timelines (packed back to back, align 1): the scan's
    # piece-parallel path with head groups (a sub-range's first <= 3 tokens up to a 16-byte boundary)
    import workloads as W
    ubig = _tile(W.config3().subset(np.arange(snap.n), align=1), 16)
    ureq = A.requests_to(ubig, device=dev)
    u_ms = []
    with torch.cuda.stream(stream):
        for k in range(max(args.warmup, 3) + 10):
            flush.zero_()
            qctx.qoe_eval(ureq, ubig.n, ubig.now_us + ubig.horizon_us, A.ANDES_EVAL_INFLIGHT, stream=stream)
            st = qctx.profile_read()
            if k >= max(args.warmup, 3):
                u_ms.append(st)
    u_scan = statistics.median([s_[1] for s_ in u_ms])
    ubytes = 4 * ubig.n_tokens + 44 * ubig.n
    qoe_eval["unaligned_pool"] = {
        "path": "timelines packed back to back (align 1): the piece-parallel path with head groups on plain TMA tiles",
        "pool_tokens": ubig.n_tokens, "scan_ms": u_scan,
        "ms_per_eval": statistics.median([s_[0] + s_[1] + s_[2] for s_ in u_ms]),
        "roofline": {"kernel": "k_qoe_scan (head groups)", "bound": "hbm", "achieved": ubytes / (u_scan / 1e3) / 1e9,
                     "peak": hbm_peak, "unit": "GB/s", "frac": ubytes / (u_scan / 1e3) / 1e9 / hbm_peak,
                     "algorithmic_bytes_per_launch": ubytes}}
    del qctx, breq, ureq

    # ---- the same decision under the LQSF priority, the Appendix-A objectives (NEXT-2) and with
    # the overhead-aware refiner (NEXT-1; prefill 5000 tok/s, no swapping)
    objectives = {}
    with torch.cuda.stream(stream):
        for name, fl in (("lqsf", A.ANDES_LQSF), ("maxmin", A.ANDES_OBJ_MAXMIN), ("perfect", A.ANDES_OBJ_PERFECT),
                         ("refine", A.ANDES_REFINE)):
            kwo = dict(preempt_cap=snap.preempt_cap, flags=A.ANDES_FORCE | fl)
            for _ in range(2):
                ctx.schedule(req, n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=stream, **kwo)
            go = torch.cuda.CUDAGraph()
            with torch.cuda.graph(go, stream=stream):
                ctx.schedule(req, n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=stream, **kwo)
            ms_o = []
            for _ in range(max(3, min(args.steps, 10))):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                go.replay()
                b.record(stream)
                b.synchronize()
                ms_o.append(a.elapsed_time(b))
            sco = out.scalars.cpu().numpy().view(np.uint32)
            objectives[name] = {"ms_per_decision": statistics.median(ms_o), "B_star": int(sco[0]),
                                "realized": int(sco[1]), "n_admit": int(sco[2]), "n_preempt": int(sco[3])}
            del go

    # ---- config 4: the 2^20-request population sharded over the ranks (multi-GPU decision)
    config4 = None if args.no_sharded else sharded_decision(args, dist, rank, ws, lr, stream, flush)

    # ---- NEXT-3: the serving loop with the decision in the loop (rank 0; replicas would repeat it)
    sim = None if (args.no_sim or rank != 0) else serving_sim(args, lr, stream)

    # ---- config 5: the 1024-scenario sweep (end-of-trace QoE per scenario)
    sweep = None if args.no_sweep else sweep_run(args, dist, rank, ws, lr, stream)

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    hreq = A.requests_to(snap, pin=True)
    tau_h = torch.from_numpy(snap.tau_us.view(np.int32)).pin_memory()
    hout = ctx.alloc_decision(n, 256, pin=True)
    e2e_steps = max(3, min(args.steps, 20))
    ctx.profile_enable(False)
    with torch.cuda.stream(stream):
        for _ in range(2):
            ctx.schedule_host(hreq, n, snap.now_us, snap.horizon_us, tau_h, snap.kv_capacity, out=hout,
                              stream=stream, **kw)
        e_ms = []
        for _ in range(e2e_steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.schedule_host(hreq, n, snap.now_us, snap.horizon_us, tau_h, snap.kv_capacity, out=hout,
                              stream=stream, **kw)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
    e_total = _max_over_ranks(dist, sum(e_ms))
    hsc = hout.scalars.numpy().view(np.uint32)
    h2d = sum(t.numel() * t.element_size() for k, t in hreq.items() if t is not None) + tau_h.numel() * 4
    d2h = 32 + n + 4 * int(hsc[2]) + 4 * int(hsc[3]) + 12 * 256 + 32
    full_upload = {"value": ws * e2e_steps / (e_total / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "api": "andes_schedule_host (whole population re-uploaded every step)"}
    e2e = e2e_incremental(args, dist, snap, ws, lr, stream)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64/f64",
        "data": "synthetic (seeded ShareGPT-shaped cyclic-burst snapshot, workloads.config3; seed 1+rank)",
        "config": {"workload": WORKLOAD, "n_requests": n, "pool_tokens": snap.n_tokens,
                   "token_events": ev_tokens, "B_cap": 256, "l2": "flushed: 256 MiB write between timed steps",
                   "launch": "one CUDA graph per decision (5 kernels)", "warm_l2_ms_per_step": warm_ms,
                   "decision": {k: int(v) for k, v in zip(A.SC_NAMES, sc)}},
        "roofline": roof,
        "qoe_eval": qoe_eval,
        "objectives": objectives,
        "config4_sharded": config4,
        "config5_sweep": sweep,
        "serving_sim": sim,
        "e2e": e2e,
        "e2e_full_upload": full_upload,
        "gpu_launches": KERNELS_PER_DECISION * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(snap)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _relaunch(n):
    """--gpus N without a launcher: re-exec this command under torch.distributed.run with N
    ranks (one process per GPU, rendezvous on 127.0.0.1), as the driver itself would."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true", help="skip the config-4 sharded decision")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 scenario sweep")
    ap.add_argument("--no-sim", action="store_true", help="skip the NEXT-3 serving-loop simulation")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
