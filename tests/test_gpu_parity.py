"""Parity of the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Bars: S_delay / S_whole exact (int64); QoE fp64 bit-equal and the
fp32 QoE within 1e-5 relative (BASELINE north star); gains fp64 bit-equal; priority keys
fp32 bit-equal; decisions (B*, serve set, admit and preempt lists in order, V(B), k*(B),
scalars) identical.  Sizes span many 4096-token scan tiles with ragged tails, empty and
degenerate cases, and the full BASELINE configurations (sampled where the oracle is slow).
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


@pytest.fixture(scope="module")
def ctx(A):
    return A.Context(max_requests=1 << 17, max_B=256, max_tokens=1 << 24, max_running=4096)


def _dev(A, snap):
    return A.requests_to(snap)


def _tau(snap):
    return torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()


# ---------------------------------------------------------------- S1 QoE
def _check_qoe(A, ctx, orc, snap, eval_time, final):
    q, q64, sd, sw, m = ctx.qoe_eval(_dev(A, snap), snap.n, eval_time,
                                     A.ANDES_EVAL_FINAL if final else A.ANDES_EVAL_INFLIGHT)
    torch.cuda.synchronize()
    oq, osd, osw, om = orc.qoe_eval(snap, eval_time, final=final)
    np.testing.assert_array_equal(m.cpu().numpy().view(np.uint32), om)
    np.testing.assert_array_equal(sd.cpu().numpy(), osd)
    np.testing.assert_array_equal(sw.cpu().numpy(), osw)
    np.testing.assert_array_equal(q64.cpu().numpy(), oq)  # bit-equal fp64
    qf = q.cpu().numpy()
    assert np.all(np.abs(qf.astype(np.float64) - oq) <= 1e-5 * np.maximum(np.abs(oq), 1e-30) + 1e-30)


@pytest.mark.parametrize("seed", range(30))
def test_qoe_random_small(A, ctx, orc, seed):
    # odd seeds: unaligned pools (the scan's general path); even seeds: 16-byte aligned timelines
    snap = W.random_small(seed, align=[4, 1][seed % 2], n=int(np.random.default_rng(seed).integers(1, 40)), max_tokens=300)
    for final in (False, True):
        _check_qoe(A, ctx, orc, snap, snap.now_us + snap.horizon_us, final)
        _check_qoe(A, ctx, orc, snap, snap.now_us, final)


def test_qoe_outputs_subset(A, ctx, orc):
    """qoe_eval(outputs=...): only the requested outputs are written (the others NULL in
    AndesQoeOut, None in Python), equal to the full call's and to the oracle's."""
    snap = W.random_small(5, n=40, max_tokens=300)
    ev = snap.now_us + snap.horizon_us
    full = ctx.qoe_eval(_dev(A, snap), snap.n, ev, A.ANDES_EVAL_INFLIGHT)
    oq, osd, osw, om = orc.qoe_eval(snap, ev, final=False)
    for outs in (("q",), ("q64", "m"), ("s_delay", "s_whole")):
        part = ctx.qoe_eval(_dev(A, snap), snap.n, ev, A.ANDES_EVAL_INFLIGHT, outputs=outs)
        torch.cuda.synchronize()
        for k, (a, b) in enumerate(zip(part, full)):
            if A.Context._QOE_OUTPUTS[k] in outs:
                np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
            else:
                assert a is None
    np.testing.assert_array_equal(full[1].cpu().numpy(), oq)
    np.testing.assert_array_equal(full[2].cpu().numpy(), osd)
    with pytest.raises(ValueError):
        ctx.qoe_eval(_dev(A, snap), snap.n, ev, outputs=("qoe",))


def test_qoe_many_tiles_ragged(A, ctx, orc):
    # ~4.7 tiles of tokens, a 100k-token request spanning many tiles, empty requests, a ragged tail
    rng = np.random.default_rng(99)
    snap = W.random_small(7, n=60, max_tokens=2000)
    snap_u = W.random_small(7, n=60, max_tokens=2000, align=1)
    long = W.snapshot(300, seed=3)
    for s in (snap, snap_u, long):
        _check_qoe(A, ctx, orc, s, s.now_us + s.horizon_us, False)
        _check_qoe(A, ctx, orc, s, s.now_us, True)
    # one request with 100,003 tokens on time then late, plus neighbours with 0 and 1 tokens
    P, ttft = 1000, 5000
    g = 100_003
    d = ttft + np.arange(g, dtype=np.int64) * P + np.where(np.arange(g) > 50_000, 7_777, 0)
    d = np.maximum.accumulate(d + rng.integers(-900, 900, g)).astype(np.uint32)
    tl = [np.zeros(0, np.uint32), d, np.array([12], np.uint32), np.zeros(0, np.uint32)]
    for align in (4, 1):
        _check_long_request(A, ctx, orc, tl, ttft, P, d, align)


def _check_long_request(A, ctx, orc, tl, ttft, P, d, align):
    gg, base, pool = W._pack(tl, align)
    n = 4
    big = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, ttft, np.uint32),
                     period_us=np.full(n, P, np.uint32), ctx_len=np.ones(n, np.uint32), n_deliv=gg,
                     max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                     rank=np.arange(n, dtype=np.uint32), running=np.zeros(n, np.uint8), tl_base=base,
                     tl_pool=pool, now_us=int(d[-1]) + 10, horizon_us=2_000_000)
    for final in (False, True):
        _check_qoe(A, ctx, orc, big, big.now_us + 3_000_000, final)
        _check_qoe(A, ctx, orc, big, big.now_us - 40_000_000, final)


@pytest.mark.parametrize("lb_ns", ["20000", "0", "1000"])
def test_qoe_long_lookback(A, orc, lb_ns, monkeypatch):
    # long requests: nearly every tile's carry comes by look-back; ANDES_LOOKBACK_NS=0 forces the
    # direct fallback on every look-back, 1000 mixes both (whichever wins, the values are equal)
    monkeypatch.setenv("ANDES_LOOKBACK_NS", lb_ns)
    c2 = A.Context(max_requests=1024, max_B=256, max_tokens=1 << 23)
    for align in (4, 1):
        snap = W.long_requests(5, align=align)
        for final in (False, True):
            _check_qoe(A, c2, orc, snap, snap.now_us, final)
            _check_qoe(A, c2, orc, snap, snap.now_us // 2, final)


@pytest.mark.parametrize("lb_ns", ["20000", "0"])
def test_schedule_long_requests(A, orc, lb_ns, monkeypatch):
    # decisions over long-output requests (the scan's look-back and its direct fallback feed
    # Q_wait and the gains): B = 1..16, M tight enough that Algorithm 1 stops early
    import dataclasses
    monkeypatch.setenv("ANDES_LOOKBACK_NS", lb_ns)
    c2 = A.Context(max_requests=1024, max_B=16, max_tokens=1 << 22)
    for seed, align in ((11, 4), (12, 1)):
        snap = W.long_requests(seed, n=40, lo=5_000, hi=12_000, align=align)
        snap = dataclasses.replace(snap, tau_us=W.tau_table(B_cap=16), kv_capacity=20_000,
                                   now_us=snap.now_us // 2, preempt_cap=3)
        _check_sched(A, c2, orc, snap)


def test_qoe_config3_full(A, ctx, orc):
    snap = W.config3()
    # the oracle is fast enough for QoE (one walk per request)
    _check_qoe(A, ctx, orc, snap, snap.now_us + snap.horizon_us, False)
    _check_qoe(A, ctx, orc, snap, snap.now_us, True)


def test_qoe_config3_unaligned(A, ctx, orc):
    """Config 3 with its timelines packed back to back (a tracker that does not pad): every
    request starts at an arbitrary token, so the scan's piece-parallel path runs with head groups
    (and the row path on the tiles that look back)."""
    snap = W.config3().subset(np.arange(65536), align=1)
    assert np.any(snap.tl_base.astype(np.int64) % 4 != 0)
    _check_qoe(A, ctx, orc, snap, snap.now_us + snap.horizon_us, False)
    _check_qoe(A, ctx, orc, snap, snap.now_us, True)


def test_schedule_config2_unaligned(A, ctx, orc):
    snap = W.config2().subset(np.arange(W.config2().n), align=1)
    _check_sched(A, ctx, orc, snap)
    _check_sched(A, ctx, orc, snap, cap=16)


# ---------------------------------------------------------------- S3 gains
def _check_gains(A, ctx, orc, snap, B_list, sub=None):
    gain, key, qw = ctx.gain_estimate(_dev(A, snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), B_list)
    torch.cuda.synchronize()
    gain, key, qw = gain.cpu().numpy(), key.cpu().numpy(), qw.cpu().numpy()
    if sub is not None:
        gain, key, qw = gain[:, sub], key[:, sub], qw[sub]
        snap = snap.subset(sub)
    og, ok, oqw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, B_list)
    np.testing.assert_array_equal(qw, oqw)
    np.testing.assert_array_equal(gain, og)
    np.testing.assert_array_equal(key.view(np.uint32), ok.view(np.uint32))


@pytest.mark.parametrize("seed", range(40))
def test_gains_random_small(A, ctx, orc, seed):
    snap = W.random_small(seed, n=int(np.random.default_rng(seed + 1).integers(1, 30)), max_tokens=200,
                          align=[4, 1][seed % 2])
    _check_gains(A, ctx, orc, snap, np.arange(1, snap.tau_us.size + 1))


def test_gains_config2_full(A, ctx, orc):
    snap = W.config2()
    _check_gains(A, ctx, orc, snap, np.arange(1, 257))


def test_gains_config3_sampled(A, ctx, orc):
    snap = W.config3()
    rng = np.random.default_rng(0)
    sub = np.sort(rng.choice(snap.n, 600, replace=False))
    _check_gains(A, ctx, orc, snap, np.array([1, 2, 3, 64, 127, 128, 200, 234, 235, 236, 255, 256]), sub)


# ---------------------------------------------------------------- S0-S6 decisions
def _run_sched(A, ctx, snap, flags=1, cap=None, cur_latency=0, prefill=5000, swap=0):
    cap = snap.preempt_cap if cap is None else cap
    d = ctx.schedule(_dev(A, snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), snap.kv_capacity,
                     preempt_cap=cap, cur_latency_us=cur_latency, flags=flags, prefill_tok_s=prefill,
                     swap_tok_s=swap)
    torch.cuda.synchronize()
    sc = d.scalars.cpu().numpy().view(np.uint32)
    return dict(mask=d.serve_mask.cpu().numpy()[:snap.n], admit=d.admit.cpu().numpy().view(np.uint32)[:sc[2]],
                preempt=d.preempt.cpu().numpy().view(np.uint32)[:sc[3]], sc=sc, V=d.V.cpu().numpy(),
                kstar=d.kstar.cpu().numpy().view(np.uint32))


def _check_sched(A, ctx, orc, snap, flags=1, cap=None, cur_latency=0, prefill=5000, swap=0):
    cap = snap.preempt_cap if cap is None else cap
    g = _run_sched(A, ctx, snap, flags, cap, cur_latency, prefill, swap)
    o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity, preempt_cap=cap,
                     cur_latency_us=cur_latency, flags=flags, prefill_tok_s=prefill, swap_tok_s=swap)
    trig = bool(g["sc"][6] & 1)
    assert trig == (o.status == 0)
    np.testing.assert_array_equal(g["mask"], o.serve_mask)
    if trig:
        assert [int(x) for x in g["sc"][[0, 1, 2, 3, 4, 5, 7]]] == [o.B_star, o.realized, o.admit.size,
                                                                    o.preempt.size, o.B_lo, o.B_hi, o.k_star]
        assert int(g["sc"][6]) & 39 == o.flags & 39  # triggered, cap hit, cap overridden, refined
        np.testing.assert_array_equal(g["admit"], o.admit)
        np.testing.assert_array_equal(g["preempt"], o.preempt)
        np.testing.assert_array_equal(g["V"], o.V)
        np.testing.assert_array_equal(g["kstar"], o.kstar)
    return g, o


def test_golden_g1_on_gpu(A, ctx, orc):
    from test_oracle_pins import g1_snapshot
    for cap in (W.UINT32_MAX, 0, 1):
        snap, d = g1_snapshot(cap)
        g, o = _check_sched(A, ctx, orc, snap, cap=cap)
        assert int(g["sc"][0]) == d["expected"]["B_star"]
        assert g["V"][:3].tolist() == d["expected"]["V_by_B"][:3]


@pytest.mark.parametrize("seed", range(60))
def test_schedule_random_small(A, ctx, orc, seed):
    snap = W.random_small(seed, B_cap=int(np.random.default_rng(seed).integers(1, 20)), align=[4, 1][seed % 2])
    flags = [1, 3, 0, 2][seed % 4]
    _check_sched(A, ctx, orc, snap, flags=flags, cur_latency=[0, 400_000][seed % 2])


def test_schedule_ties_and_zero_gains(A, ctx, orc):
    # every request on schedule far ahead -> all gains 0: selection by rank only
    n = 300
    tl = [np.arange(50, dtype=np.uint32) * 1000 for _ in range(n)]
    g, base, pool = W._pack(tl)
    rng = np.random.default_rng(5)
    snap = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                      period_us=np.full(n, 200_000, np.uint32), ctx_len=rng.integers(1, 40, n).astype(np.uint32),
                      n_deliv=g, max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=rng.permutation(n).astype(np.uint32), running=(rng.random(n) < 0.3).astype(np.uint8),
                      tl_base=base, tl_pool=pool, now_us=1_000_000, horizon_us=2_000_000,
                      tau_us=W.tau_table(64), kv_capacity=900)
    for cap in (W.UINT32_MAX, 0, 3):
        _check_sched(A, ctx, orc, snap, cap=cap)


def test_schedule_config2_full(A, ctx, orc):
    snap = W.config2()
    _check_sched(A, ctx, orc, snap)
    _check_sched(A, ctx, orc, snap, flags=3)
    _check_sched(A, ctx, orc, snap, cap=16)


def test_schedule_config3_properties(A, ctx, orc):
    """Full-size config 3 (the bench workload, same launch): the oracle needs minutes, so check
    (a) determinism, (b) B* / serve set against Algorithm 1 recomputed on host from the GPU's
    gain_estimate keys at B*, whose parity is sampled in test_gains_config3_sampled, (c) the cap."""
    snap = W.config3()
    g1 = _run_sched(A, ctx, snap)
    g2 = _run_sched(A, ctx, snap)
    for k in g1:
        np.testing.assert_array_equal(g1[k], g2[k])
    sc = g1["sc"]
    Bs, ks = int(sc[0]), int(sc[7])
    assert sc[6] & 1 and 1 <= Bs <= 256 and sc[5] == 256
    gain, key, qw = ctx.gain_estimate(_dev(A, snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), [Bs])
    key = key.cpu().numpy()[0]
    gain = gain.cpu().numpy()[0]
    order = np.lexsort((snap.rank, -key.astype(np.float64)))
    csum = np.cumsum(snap.ctx_len[order].astype(np.int64))
    k = int(min(Bs, np.searchsorted(csum, snap.kv_capacity, side="right")))
    assert k == ks
    S = set(order[:k].tolist())
    vfix = int(np.sum(np.rint(gain[order[:k]] * 2.0 ** 32).astype(np.int64)))
    assert vfix == int(g1["V"][Bs - 1])
    assert int(np.max(g1["V"])) == int(g1["V"][Bs - 1])
    running = set(np.nonzero(snap.running)[0].tolist())
    victims = running - S
    assert int(sc[3]) == min(len(victims), snap.preempt_cap) or sc[6] & 4
    assert set(g1["preempt"].tolist()) <= victims


def test_schedule_host_path_matches(A, ctx, orc):
    snap = W.config2()
    g = _run_sched(A, ctx, snap, cap=16)
    hreq = A.requests_to(snap, pin=True)
    tau_h = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).pin_memory()
    out, rc = ctx.schedule_host(hreq, snap.n, snap.now_us, snap.horizon_us, tau_h, snap.kv_capacity,
                                preempt_cap=16)
    sc = out.scalars.numpy().view(np.uint32)
    np.testing.assert_array_equal(sc, g["sc"])
    np.testing.assert_array_equal(out.serve_mask.numpy()[:snap.n], g["mask"])
    np.testing.assert_array_equal(out.preempt.numpy().view(np.uint32)[:sc[3]], g["preempt"])


def test_not_triggered(A, ctx, orc):
    snap = W.random_small(4, n=10)
    snap.kv_capacity = 10_000
    _check_sched(A, ctx, orc, snap, flags=0, cur_latency=0)


def _snap_from(tl, *, P=208_333, ttft=1_000_000, l=None, running=None, now=3_000_000, horizon=2_000_000,
               B_cap=8, M=10_000, rank=None, align=4):
    n = len(tl)
    g, base, pool = W._pack([np.asarray(t, np.uint32) for t in tl], align)
    return W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, ttft, np.uint32),
                      period_us=np.full(n, P, np.uint32),
                      ctx_len=np.asarray(l if l is not None else np.full(n, 100), np.uint32), n_deliv=g,
                      max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=np.asarray(rank if rank is not None else np.arange(n), np.uint32),
                      running=np.asarray(running if running is not None else np.zeros(n), np.uint8),
                      tl_base=base, tl_pool=pool, now_us=now, horizon_us=horizon, tau_us=W.tau_table(B_cap),
                      kv_capacity=M)


def test_schedule_degenerate_cases(A, ctx, orc):
    """The degenerate inputs of the decision, each against the oracle: one request; no request
    has a token; B_cap = 1; every request running with the running set over M (the cap is
    overridden by memory, O9); M fits exactly one request; a preemption cap of 0; identical
    requests that differ only in rank (ties broken by rank, R10)."""
    late = [np.arange(6) * 250_000 + 1_400_000]
    cases = [
        (_snap_from(late), {}),
        (_snap_from(late, running=[1]), {}),
        (_snap_from([[], [], []]), {}),
        (_snap_from(late * 5, B_cap=1), {}),
        (_snap_from(late * 6, running=[1] * 6, l=[3000] * 6, M=10_000), {"cap": 2}),
        (_snap_from(late * 6, running=[1, 1, 0, 0, 0, 0], l=[5000] * 6, M=5000), {"cap": 0}),
        (_snap_from(late * 7, rank=[6, 5, 4, 3, 2, 1, 0], B_cap=3), {"cap": 1}),
        (_snap_from(late * 4 + [[]] * 4, running=[0, 1] * 4, l=[100, 200, 300, 400] * 2, B_cap=8), {"cap": 0}),
    ]
    for snap, kw in cases:
        for flags in (1, 1 | 16, 1 | 2):
            _check_sched(A, ctx, orc, snap, flags=flags, **kw)


# ---------------------------------------------------------------- config 1: 200-iteration driver
def test_config1_iteration_driver(A, ctx, orc):
    """BASELINE config 1 (tests/config1.py): on every iteration the GPU decision equals the
    oracle's, and at every candidate B Algorithm 2 on the GPU (andes_knapsack_dp) equals brute
    force and bounds Algorithm 1 from above (SPEC acceptance #2/#3)."""
    from config1 import QualityTracker, run
    NEG = -(1 << 63)

    def gpu_dp(q, l, B, M):
        x, best, Vb = ctx.knapsack_dp(torch.tensor(q, dtype=torch.int64, device="cuda"),
                                      torch.tensor(l, dtype=torch.int32, device="cuda"), B, M)
        torch.cuda.synchronize()
        b = int(best.item())
        return (None if b == NEG else b), [None if int(v) == NEG else int(v) for v in Vb.cpu().numpy()]

    qt = QualityTracker(orc, exact_dp=gpu_dp)

    def decide(snap):
        return _check_sched(A, ctx, orc, snap, flags=1)[1]

    assert run(decide, on_iter=qt) >= 150
    assert qt.summary()["B_values_checked"] >= 150


def test_schedule_survivor_overflow_fallback(A, ctx, orc):
    """More survivors than the pruned path holds (identical late requests: every bound ties, so
    every request survives): k_select evaluates every request at its B and radix-selects
    (ANDES_F_SLOW_PATH); the decision must still equal the oracle's."""
    n = 3500
    tl = [(np.arange(6, dtype=np.uint32) * 250_000 + 1_400_000) for _ in range(n)]
    g, base, pool = W._pack(tl)
    rng = np.random.default_rng(11)
    snap = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                      period_us=np.full(n, 208_333, np.uint32), ctx_len=np.full(n, 100, np.uint32),
                      n_deliv=g, max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=rng.permutation(n).astype(np.uint32), running=(rng.random(n) < 0.02).astype(np.uint8),
                      tl_base=base, tl_pool=pool, now_us=3_000_000, horizon_us=2_000_000,
                      tau_us=W.tau_table(48), kv_capacity=4000)
    gg, o = _check_sched(A, ctx, orc, snap, cap=5)
    assert int(gg["sc"][6]) & A.ANDES_F_SLOW_PATH
    # max-min: every request has the same non-zero key (Q_min - Q_wait > 0, equal l): the
    # fallback, with one sorted list shared by all B; perfect count: every gain is exactly 0,
    # so the exact-zero rank cut keeps the pruned path
    gg, o = _check_sched(A, ctx, orc, snap, flags=1 | 32, cap=5)
    assert int(gg["sc"][6]) & A.ANDES_F_SLOW_PATH
    gg, o = _check_sched(A, ctx, orc, snap, flags=1 | 64, cap=5)
    assert not int(gg["sc"][6]) & A.ANDES_F_SLOW_PATH


def test_schedule_exact_zero_rank_pruning(A, ctx, orc):
    """Most requests are ahead of schedule (no undelivered due token: gain exactly 0 at every B),
    so the key bucket holding theta is the zero bucket; k_compact keeps only the B_hi smallest
    ranks of the exact zeros (the survivors then fit: no slow path), and the decision, the
    zero-gain requests it takes included (Algorithm 1 takes gain-0 requests while they fit),
    must equal the oracle's."""
    n, nz = 5000, 4880
    rng = np.random.default_rng(5)
    tl = []
    for i in range(n):
        if i < nz:  # 60 tokens delivered right after ttft: far ahead of the 208 ms schedule
            tl.append((1_000_000 + np.arange(60, dtype=np.uint32) * 1_000).astype(np.uint32))
        else:  # behind: 6 tokens, late
            tl.append((np.arange(6, dtype=np.uint32) * 250_000 + 1_400_000 + rng.integers(0, 90_000)).astype(np.uint32))
    g, base, pool = W._pack(tl)
    perm = rng.permutation(n)
    snap = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                      period_us=np.full(n, 208_333, np.uint32), ctx_len=rng.integers(50, 400, n).astype(np.uint32),
                      n_deliv=g, max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=perm.astype(np.uint32), running=(rng.random(n) < 0.01).astype(np.uint8),
                      tl_base=base, tl_pool=pool, now_us=3_000_000, horizon_us=2_000_000,
                      tau_us=W.tau_table(200), kv_capacity=30_000)
    for flags in (1, 1 | 16, 1 | 32):
        gg, o = _check_sched(A, ctx, orc, snap, flags=flags, cap=4)
        assert not (int(gg["sc"][6]) & A.ANDES_F_SLOW_PATH), flags


# ---------------------------------------------------------------- config-5 sweep: scenario means
def test_scenario_means_match_oracle(A, ctx, orc):
    """andes_qoe_scenario_mean vs the oracle: FINAL-mode QoE per request (R19), mean over g >= 1
    per scenario.  Counts exact; means within 1e-12 relative of the exact (fsum) mean."""
    import math
    scen = [(1, 0.5), (2, 1.0), (3, 2.05), (4, 1.5), (5, 0.75)]
    snap, off = W.sweep(scen, n_base=60)
    # an empty scenario and a scenario whose requests have no tokens
    off = np.concatenate([off[:2], off[1:2], off[2:]]).astype(np.uint32)
    mean, cnt = ctx.qoe_scenario_mean(_dev(A, snap), snap.n, torch.from_numpy(off.view(np.int32)).cuda())
    torch.cuda.synchronize()
    mean, cnt = mean.cpu().numpy(), cnt.cpu().numpy()
    q, sd, sw, m = orc.qoe_eval(snap, 0, final=True)
    for s in range(off.size - 1):
        sel = np.arange(off[s], off[s + 1])
        sel = sel[snap.n_deliv[sel] >= 1]
        assert int(cnt[s]) == sel.size
        exact = math.fsum(q[sel]) / sel.size if sel.size else 0.0
        assert abs(mean[s] - exact) <= 1e-12 * max(1.0, abs(exact)), (s, mean[s], exact)


# ---------------------------------------------------------------- LQSF priority (NEXT-2, reading R21)
@pytest.mark.parametrize("seed", range(20))
def test_schedule_lqsf_random_small(A, ctx, orc, seed):
    snap = W.random_small(seed + 100, B_cap=int(np.random.default_rng(seed).integers(1, 20)), align=[4, 1][seed % 2])
    _check_sched(A, ctx, orc, snap, flags=[1 | 16, 3 | 16][seed % 2], cap=[W.UINT32_MAX, 1][seed % 2])


def test_schedule_lqsf_config2(A, ctx, orc):
    snap = W.config2()
    g, o = _check_sched(A, ctx, orc, snap, flags=1 | 16, cap=16)
    g2, o2 = _check_sched(A, ctx, orc, snap, flags=1, cap=16)
    assert not np.array_equal(g["V"], g2["V"])  # the priority changed the decision


# ---------------------------------------------------------------- Appendix-A objectives (R22-R23)
@pytest.mark.parametrize("seed", range(24))
def test_schedule_objectives_random_small(A, ctx, orc, seed):
    snap = W.random_small(seed + 200, B_cap=int(np.random.default_rng(seed).integers(1, 20)), align=[4, 1][seed % 2])
    obj = [32, 64][seed % 2]
    extra = [0, 16, 2][seed % 3]  # plain, with the LQSF priority, with pruning
    _check_sched(A, ctx, orc, snap, flags=1 | obj | extra, cap=[W.UINT32_MAX, 1, 0][seed % 3])


def test_schedule_objectives_g1_and_config2(A, ctx, orc):
    from test_oracle_pins import g1_snapshot
    snap, d = g1_snapshot()
    for obj in (32, 64):
        _check_sched(A, ctx, orc, snap, flags=1 | obj)
    snap = W.config2()
    for obj in (32, 64):
        _check_sched(A, ctx, orc, snap, flags=1 | obj, cap=16)


# ---------------------------------------------------------------- overhead-aware refiner (NEXT-1)
def test_refiner_g1_on_gpu(A, ctx, orc):
    from test_oracle_pins import g1_snapshot
    snap, d = g1_snapshot()
    for prefill in (20, 40, 0):
        g, o = _check_sched(A, ctx, orc, snap, flags=1 | 128, prefill=prefill)
    g, o = _check_sched(A, ctx, orc, snap, flags=1 | 128, prefill=20)
    assert g["admit"].tolist() == [] and g["preempt"].tolist() == [] and g["sc"][6] & 32


@pytest.mark.parametrize("seed", range(24))
def test_refiner_random_small(A, ctx, orc, seed):
    rng = np.random.default_rng(seed + 7)
    snap = W.random_small(seed + 300, B_cap=int(rng.integers(1, 20)), align=[4, 1][seed % 2])
    prefill = int([0, 30, 200, 5000, 100000][seed % 5])
    swap = int([0, 0, 400, 0, 50][seed % 5])
    extra = [0, 16, 32][seed % 3]
    _check_sched(A, ctx, orc, snap, flags=1 | 128 | extra, cap=[W.UINT32_MAX, 2][seed % 2], prefill=prefill,
                 swap=swap)


def test_refiner_config2(A, ctx, orc):
    snap = W.config2()
    for prefill, swap in ((5000, 0), (500, 20000), (50_000, 0)):
        _check_sched(A, ctx, orc, snap, flags=1 | 128, cap=16, prefill=prefill, swap=swap)


# ---------------------------------------------------------------- Algorithm 2 on the GPU (NEXT-4)
@pytest.mark.parametrize("seed", range(16))
def test_knapsack_dp_matches_algorithm2(A, ctx, seed):
    """andes_knapsack_dp vs the oracle's line-by-line transcription of Algorithm 2 (exact integer
    values): the same optimum, the same solution vector (tie rules included), and per-b optima
    equal to brute force."""
    from oracle import exact as X
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 12))
    B = int(rng.integers(0, n + 2))
    M = int(rng.integers(0, 60))
    l = rng.integers(1, 25, n).tolist()
    q = (rng.integers(-5, 12, n) * (2 ** 28 if seed % 2 else 1)).tolist()  # ties and negatives
    if seed % 4 == 0:
        q = [3] * n  # all tied
    x, best, Vb = ctx.knapsack_dp(torch.tensor(q, dtype=torch.int64, device="cuda"),
                                  torch.tensor(l, dtype=torch.int32, device="cuda"), B, M)
    torch.cuda.synchronize()
    qm, xo = X.dp_algorithm2(q, l, B, M)
    if qm is None:
        assert int(best.item()) == -(1 << 63)
    else:
        assert int(best.item()) == qm
        assert x.cpu().numpy().tolist() == xo
    for b in range(B + 1):
        bf = X.brute_force(q, l, b, M)[0]
        v = int(Vb[b].item())
        assert (v == -(1 << 63) and bf is None) or v == bf, (b, v, bf)


def test_knapsack_dp_bounds_the_greedy_on_a_snapshot(A, ctx, orc):
    """Decision-quality reference: at every B the exact optimum of Eq. 5 (Algorithm 2 on the GPU
    over the oracle's gains in 2^-32 units) is >= Algorithm 1's V(B) from andes_schedule."""
    snap = W.random_small(21, n=14, B_cap=6)
    g = _run_sched(A, ctx, snap, flags=1)
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, np.arange(1, 7))
    l = torch.from_numpy(snap.ctx_len.astype(np.int32)).cuda()
    for B in range(int(g["sc"][4]), int(g["sc"][5]) + 1):
        q = torch.from_numpy(np.rint(gain[B - 1] * 2.0 ** 32).astype(np.int64)).cuda()
        x, best, Vb = ctx.knapsack_dp(q, l, B, snap.kv_capacity)
        torch.cuda.synchronize()
        exact = max(int(v) for v in Vb.cpu().numpy()[: B + 1] if v != -(1 << 63))
        assert exact >= int(g["V"][B - 1])


# ---------------------------------------------------------------- two-tile scan units
_TW2_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2404_16283_b200 as A, workloads as W, oracle
from test_gpu_parity import _check_qoe, _check_sched
oracle.build()
ctx = A.Context(max_requests=1 << 17, max_B=256, max_tokens=1 << 24, max_running=4096)
for seed in range(16):
    snap = W.random_small(seed, align=[4, 1][seed % 2], n=int(np.random.default_rng(seed).integers(1, 40)), max_tokens=300)
    for final in (False, True):
        _check_qoe(A, ctx, oracle, snap, snap.now_us + snap.horizon_us, final)
for align in (4, 1):
    snap = W.long_requests(5, align=align)
    for final in (False, True):
        _check_qoe(A, ctx, oracle, snap, snap.now_us, final)
snap = W.config3()
_check_qoe(A, ctx, oracle, snap, snap.now_us + snap.horizon_us, False)
_check_sched(A, ctx, oracle, W.config2(), cap=16)
# the three carry cases of the two-tile pass-2 skip (scan.cu, warp_tile_aligned): timelines
# delivered ahead of consumption (clamped at t), late then faster than the period (the carry
# dominates: closed form), lateness oscillating by +-P (the zero-carry lateness catches up inside
# a sub-range: partial walk), slowly growing lateness with jitter
rng = np.random.default_rng(7)
n = 96
P = rng.choice([20_000, 50_000, 208_333], n).astype(np.int64)
ttft = rng.choice([0, 1_000_000], n).astype(np.int64)
tls = []
for i in range(n):
    g = int(rng.integers(1, 6000))
    j = np.arange(g, dtype=np.int64)
    kind = i % 4
    if kind == 0:
        d = ttft[i] + j * (P[i] // 4)
    elif kind == 1:
        d = ttft[i] + 5 * P[i] + j * (P[i] * 3 // 4)
    elif kind == 2:
        d = ttft[i] + j * P[i] + rng.integers(-P[i], P[i] + 1, g)
    else:
        d = ttft[i] + j * (P[i] * 11 // 10) + rng.integers(-P[i] // 3, P[i] // 3 + 1, g)
    tls.append(np.maximum.accumulate(np.maximum(d, 0)).astype(np.uint32))
# each request evaluated shortly after its last delivery (its late tokens then clamp at t)
now = 1 << 31
arr = np.array([now - int(t[-1]) - int(rng.integers(0, 2 * P[i])) for i, t in enumerate(tls)], np.int64)
for align in (4, 1):
    g, base, pool = W._pack(tls, align)
    snap = W.Snapshot(arrival_us=arr, ttft_us=ttft.astype(np.uint32), period_us=P.astype(np.uint32),
                      ctx_len=rng.integers(1, 4096, n).astype(np.uint32), n_deliv=g,
                      max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=np.arange(n, dtype=np.uint32), running=np.zeros(n, np.uint8), tl_base=base, tl_pool=pool,
                      now_us=now, horizon_us=2_000_000)
    for ev in (snap.now_us, snap.now_us + snap.horizon_us):
        _check_qoe(A, ctx, oracle, snap, ev, False)
    _check_qoe(A, ctx, oracle, snap, snap.now_us, True)
print("tw2 ok")
"""


@pytest.mark.parametrize("tw", ["2", "1"])
def test_scan_unit_width_forced(tw):
    """The scan's work unit is two warp-tiles (2048 tokens) on large pools and one on small ones;
    ANDES_SCAN_TW forces either, so both are checked against the oracle on the same inputs
    (aligned and unaligned pools, long requests, config 3, a config-2 decision, and timelines
    built for the three carry cases of the two-tile pass-2 skip)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ANDES_SCAN_TW=tw)
    r = subprocess.run([sys.executable, "-c", _TW2_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "tw2 ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_refiner_fig7_toy_on_gpu(A, ctx, orc):
    """The constructed Fig. 7 scenario (test_oracle_pins.fig7_snapshot) through the
    C ABI: admits {R9, R10}, preempts {R1, R2} after refinement, equal to the oracle, also with
    swapping available and with cheap admissions (every pair kept)."""
    from test_oracle_pins import fig7_snapshot
    snap = fig7_snapshot()
    g, o = _check_sched(A, ctx, orc, snap, flags=1 | 128, prefill=50)
    assert (g["admit"] + 1).tolist() == [10, 9] and (g["preempt"] + 1).tolist() == [1, 2]
    g, o = _check_sched(A, ctx, orc, snap, flags=1 | 128, prefill=200)
    assert (g["admit"] + 1).tolist() == [10, 9, 8]
    for prefill, swap in ((50, 100), (50, 1000), (25, 400)):
        _check_sched(A, ctx, orc, snap, flags=1 | 128, prefill=prefill, swap=swap)


# ---------------------------------------------------------------- maximum sizes
def _many_short(n, seed, run_frac, l_lo, l_hi, M):
    """n requests with short, partly late timelines and small contexts (B_hi reaches B_cap)."""
    rng = np.random.default_rng(seed)
    tl = []
    for i in range(n):
        g = int(rng.integers(0, 12))
        d = 1_000_000 + np.arange(g) * 200_000 + rng.integers(0, 900_000)
        tl.append(np.maximum.accumulate(np.minimum(d, 4_900_000)).astype(np.uint32))
    g, base, pool = W._pack(tl)
    return W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                      period_us=rng.choice([208_333, 303_030], n).astype(np.uint32),
                      ctx_len=rng.integers(l_lo, l_hi, n).astype(np.uint32), n_deliv=g,
                      max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=rng.permutation(n).astype(np.uint32), running=(rng.random(n) < run_frac).astype(np.uint8),
                      tl_base=base, tl_pool=pool, now_us=5_000_000, horizon_us=2_000_000, kv_capacity=M)


def test_schedule_max_B_cap_1024(A, orc):
    """B_cap at the library's maximum (1024 candidate batch sizes, 1024 k_select CTAs, Algorithm 1
    prefixes up to 1024 long): every output equal to the oracle's, with and without the cap."""
    import dataclasses
    c = A.Context(max_requests=8192, max_B=1024, max_tokens=1 << 20)
    snap = dataclasses.replace(_many_short(3000, 4, 0.1, 20, 200, 120_000), tau_us=W.tau_table(1024))
    for cap, flags in ((W.UINT32_MAX, 1), (16, 1), (16, 1 | 16)):
        g, o = _check_sched(A, c, orc, snap, flags=flags, cap=cap)
        assert o.B_hi == 1024 and int(o.kstar.max()) > 512


def test_schedule_large_running_sets(A, orc):
    """Running sets past the per-B cap staging (n_run > 512: the general staging; > 2048: the
    last CTA's general finalize) up to the 4096 maximum, against the oracle."""
    c = A.Context(max_requests=8192, max_B=256, max_tokens=1 << 20)
    for n, frac, cap in ((1500, 0.6, 16), (5000, 0.55, 40), (5000, 0.8, W.UINT32_MAX)):
        snap = _many_short(n, n + int(frac * 100), frac, 1, 40, 200_000)
        assert int(snap.running.sum()) <= 4096
        g, o = _check_sched(A, c, orc, snap, cap=cap)
        assert not int(g["sc"][6]) & A.ANDES_F_TRUNCATED
