"""Multi-GPU decision (andes_schedule_shard) on one GPU: G shard contexts run the
five steps in lockstep and the round blocks are gathered exactly as an all-gather would (rank
order).  Pins (SURVEY 8(c) "Multi-GPU"): the sharded decision equals the CPU oracle's decision on
the concatenated population bit for bit, and equals the single-GPU decision."""
import numpy as np
import pytest
import torch

import workloads as W
from conftest import assert_decision_equal, oracle_decision_cached, snapshot_cached

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


_CTX = {}


def _ctx(A, key, n, tokens):
    c = _CTX.get(key)
    if c is None or c.limits.max_requests < n or c.limits.max_tokens < tokens:
        c = A.Context(max_requests=max(n, 1024), max_B=256, max_tokens=max(tokens + 64, 1 << 16))
        _CTX[key] = c
    return c


def _tau(snap):
    return torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()


def run_sharded(A, snap, G, cap=None, flags=1, cur_latency=0, cuts=None):
    cap = snap.preempt_cap if cap is None else cap
    n = snap.n
    cuts = np.linspace(0, n, G + 1).astype(np.int64) if cuts is None else np.asarray(cuts)
    shards = [snap.subset(np.arange(cuts[g], cuts[g + 1])) for g in range(G)]
    tau = _tau(snap)
    B_cap = int(tau.numel())
    ctxs = [_ctx(A, ("shard", g), s.n, s.n_tokens) for g, s in enumerate(shards)]
    sh = [c.shard_init(G, g, B_cap) for g, c in enumerate(ctxs)]
    bufs = [c.alloc_shard_buffers(x) for c, x in zip(ctxs, sh)]
    outs = [c.alloc_shard_decision(s.n, B_cap) for c, s in zip(ctxs, shards)]
    reqs = [A.requests_to(s) for s in shards]
    prev = [None] * G
    for step in range(A.SHARD_STEPS):
        for g in range(G):
            send = bufs[g][0][step] if step < A.SHARD_ROUNDS else None
            ctxs[g].schedule_shard(sh[g], step, reqs[g], shards[g].n, snap.now_us, snap.horizon_us, tau,
                                   snap.kv_capacity, outs[g], recv=prev[g], send=send, preempt_cap=cap,
                                   cur_latency_us=cur_latency, flags=flags)
        if step < A.SHARD_ROUNDS:
            gathered = torch.cat([bufs[g][0][step] for g in range(G)])
            for g in range(G):
                bufs[g][1][step].copy_(gathered)
            prev = [bufs[g][1][step] for g in range(G)]
    torch.cuda.synchronize()
    res = []
    for g in range(G):
        sc = outs[g].scalars.cpu().numpy().view(np.uint32).copy()
        res.append(dict(sc=sc, V=outs[g].V.cpu().numpy(), kstar=outs[g].kstar.cpu().numpy().view(np.uint32),
                        admit=outs[g].admit.cpu().numpy().view(np.uint32)[:sc[2]],
                        preempt=outs[g].preempt.cpu().numpy().view(np.uint32)[:sc[3]],
                        mask=outs[g].serve_mask.cpu().numpy()[:shards[g].n]))
    return res


def single(A, snap, cap=None, flags=1, cur_latency=0):
    cap = snap.preempt_cap if cap is None else cap
    ctx = _ctx(A, "single", snap.n, snap.n_tokens)
    d = ctx.schedule(A.requests_to(snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), snap.kv_capacity,
                     preempt_cap=cap, cur_latency_us=cur_latency, flags=flags)
    torch.cuda.synchronize()
    sc = d.scalars.cpu().numpy().view(np.uint32).copy()
    return dict(sc=sc, V=d.V.cpu().numpy(), kstar=d.kstar.cpu().numpy().view(np.uint32),
                admit=d.admit.cpu().numpy().view(np.uint32)[:sc[2]],
                preempt=d.preempt.cpu().numpy().view(np.uint32)[:sc[3]], mask=d.serve_mask.cpu().numpy()[:snap.n])


def check(A, orc, snap, G, cuts=None, name=None, **kw):
    """Sharded decision == oracle decision (every output, lists in order) and == the single-GPU
    decision.  name: a full-size snapshot whose oracle decision is cached across tests."""
    res = run_sharded(A, snap, G, cuts=cuts, **kw)
    ref = single(A, snap, **kw)
    okw = dict(cap=kw.get("cap"), flags=kw.get("flags", 1), cur_latency=kw.get("cur_latency", 0))
    if name is not None:
        o = oracle_decision_cached(orc, name, snap, **okw)
    else:
        cap = snap.preempt_cap if okw["cap"] is None else okw["cap"]
        o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity, preempt_cap=cap,
                         cur_latency_us=okw["cur_latency"], flags=okw["flags"], threads=orc.nproc())
    mask = np.concatenate([r["mask"] for r in res])
    for r in res:
        assert_decision_equal(dict(r, mask=mask), o)
    trig = bool(ref["sc"][6] & 1)
    np.testing.assert_array_equal(np.concatenate([r["mask"] for r in res]), ref["mask"])
    for r in res:
        assert bool(r["sc"][6] & 1) == trig
        if not trig:
            continue
        np.testing.assert_array_equal(r["sc"][[0, 1, 2, 3, 4, 5, 7]], ref["sc"][[0, 1, 2, 3, 4, 5, 7]])
        assert r["sc"][6] & 7 == ref["sc"][6] & 7
        np.testing.assert_array_equal(r["V"], ref["V"])
        np.testing.assert_array_equal(r["kstar"], ref["kstar"])
        np.testing.assert_array_equal(r["admit"], ref["admit"])
        np.testing.assert_array_equal(r["preempt"], ref["preempt"])
    return res, ref


@pytest.mark.parametrize("seed", range(24))
def test_shard_random_small(A, orc, seed):
    rng = np.random.default_rng(seed)
    snap = W.random_small(seed, B_cap=int(rng.integers(1, 20)))
    G = int(rng.integers(1, 6))
    check(A, orc, snap, G, flags=[1, 3, 0, 2][seed % 4], cur_latency=[0, 400_000][seed % 2],
          cap=[W.UINT32_MAX, 0, 2][seed % 3])


def test_shard_uneven_and_empty_shards(A, orc):
    snap = W.random_small(3, n=25, B_cap=12)
    check(A, orc, snap, 4, cuts=[0, 0, 3, 25, 25])
    check(A, orc, snap, 8, cuts=[0, 1, 2, 3, 4, 5, 6, 7, 25])


def test_shard_golden_g1(A, orc):
    from test_oracle_pins import g1_snapshot
    for cap in (W.UINT32_MAX, 0, 1):
        snap, d = g1_snapshot(cap)
        res, ref = check(A, orc, snap, 2, cap=cap)
        assert int(res[0]["sc"][0]) == d["expected"]["B_star"]


@pytest.mark.parametrize("G", [2, 3, 8])
def test_shard_config2(A, orc, G):
    snap = snapshot_cached("config2")
    check(A, orc, snap, G, name="config2")
    check(A, orc, snap, G, cap=16, flags=3, name="config2")


def test_shard_config3(A, orc):
    snap = snapshot_cached("config3")
    for G in (1, 2, 8):
        check(A, orc, snap, G, name="config3")


def test_shard_long_contexts_reach_the_long_bucket(A, orc):
    """Few short contexts: the B_max walk of step 1 needs the ranks' lists of their smallest
    contexts >= 4095 tokens (exact merge)."""
    snap = W.random_small(8, n=40, B_cap=16)
    rng = np.random.default_rng(2)
    snap.ctx_len[:] = rng.integers(4000, 9000, snap.n).astype(np.uint32)
    snap.kv_capacity = 60_000
    check(A, orc, snap, 3)
    check(A, orc, snap, 5, cap=1)


def test_shard_lqsf(A, orc):
    snap = snapshot_cached("config2")
    check(A, orc, snap, 3, flags=1 | 16, cap=16, name="config2")
    check(A, orc, W.random_small(5, B_cap=9), 2, flags=1 | 16)
