"""Pins for the CPU oracle (-m "not gpu").

Every check here ties oracle/andes_oracle.c to something other than itself:
worked examples from SPEC.md, closed forms of the paper's Fig. 5 cases,
an independent exact-rational walk (oracle/exact.py), brute force and
Algorithm 2 for the knapsack, and the derived golden decision G1.
"""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

import workloads as W
from oracle import exact as X

S = 1_000_000  # microseconds per second
GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- O2: worked examples
def test_spec_qoe_7_9(orc):
    # ideal [1,2,3], actual [1,2,5] (speed 1) -> S_delay 2, S_whole 9, QoE 7/9
    sd, sw, q = orc.qoe_walk([1 * S, 2 * S, 5 * S], ttft=1 * S, P=1 * S, t=0, m=0, final=True)
    assert (sd, sw) == (2 * S, 9 * S)
    assert q == 1.0 - 2.0 / 9.0
    assert abs(q - 7 / 9) < 1e-15


def test_spec_recurrence_example(orc):
    # deliveries [1.0, 3.0, 3.0], ideal [1.0, 1.5, 2.0], speed 2 -> actual [1.0, 3.0, 3.5]
    act = X.actual_consumption([1, 3, 3], X.ideal_times(1, 2, 3), 2)
    assert act == [F(1), F(3), F(7, 2)]
    sd, sw, q = orc.qoe_walk([1 * S, 3 * S, 3 * S], ttft=1 * S, P=S // 2, t=0, m=0, final=True)
    # S_delay = 0 + 1.5 + 1.5 ; S_whole = 2.5 + 2.0 + 1.5
    assert (sd, sw) == (3 * S, 6 * S)


def test_spec_ideal_timeline():
    # arrival 0, ttft 1 s, 4 tok/s -> [1.0, 1.25, 1.5]
    assert X.ideal_times(1, 4, 3) == [F(1), F(5, 4), F(3, 2)]


def test_nothing_arrives_is_zero(orc):
    # P:L319 "when no tokens arrive ... worst possible QoE of 0"; ttft 1, speed 1, t = 3 -> 0
    sd, sw, q = orc.qoe_walk([], ttft=1 * S, P=1 * S, t=3 * S, m=3)
    assert sd == sw == 3 * S and q == 0.0
    # R4: m = 0 (nothing due yet) -> S_whole = 0 -> QoE 1; exactly at T_1^Ideal -> 1; 1 us later -> 0
    assert orc.qoe_walk([], 1 * S, 1 * S, t=S - 1, m=0)[2] == 1.0
    assert orc.qoe_walk([], 1 * S, 1 * S, t=S, m=1)[2] == 1.0
    assert orc.qoe_walk([], 1 * S, 1 * S, t=S + 1, m=1)[2] == 0.0


# ---------------------------------------------------------------- O2: Fig. 5 closed forms
@pytest.mark.parametrize("n", [1, 2, 5, 17, 100])
def test_fig5a_on_time_is_one(orc, n):
    # Fig. 5a: every token no later than ideal -> QoE 1; early delivery neutral
    P, ttft = 200_000, 1_300_000
    ideal = [ttft + j * P for j in range(n)]
    early = [max(0, x - 123_457 * (j % 3)) for j, x in enumerate(ideal)]
    for D in (ideal, sorted(early)):
        sd, sw, q = orc.qoe_walk(D, ttft, P, t=0, m=0, final=True)
        assert sd == 0 and q == 1.0
        # in flight at any time after the last ideal time
        sd, sw, q = orc.qoe_walk(D, ttft, P, t=ideal[-1] + 7, m=n)
        assert sd == 0 and q == 1.0


@pytest.mark.parametrize("n,D", [(2, 1), (3, 400_000), (10, 2_500_000), (64, 37_000_001)])
def test_fig5b_ttft_missed(orc, n, D):
    # Fig. 5b: all tokens late by D, paced at s: QoE = C/(nD + C), C = n(n-1)/(2s)
    P, ttft = 300_000, 1_000_000
    s = F(S, P)  # tokens per second
    Dl = [ttft + D + j * P for j in range(n)]
    sd, sw, q = orc.qoe_walk(Dl, ttft, P, t=0, m=0, final=True)
    exp = X.qoe_ttft_missed(n, F(D, S), s)
    assert F(sd, sw) == 1 - exp if sw else True
    assert abs(q - float(exp)) < 1e-15
    assert sd == n * D and sw == n * D + P * n * (n - 1) // 2


@pytest.mark.parametrize("n", [2, 3, 9, 50])
def test_fig5c_slow_stream(orc, n):
    # Fig. 5c: first token on time, then rate r < s: QoE = s/(2s - r), any n
    P, Pr, ttft = 300_000, 500_000, 1_000_000  # s = 10/3, r = 2
    Dl = [ttft + j * Pr for j in range(n)]
    sd, sw, q = orc.qoe_walk(Dl, ttft, P, t=0, m=0, final=True)
    exp = X.qoe_slow_stream(F(S, Pr), F(S, P))
    assert exp == F(5, 7)
    assert F(S, 1) and F(sw - sd, sw) == exp
    assert abs(q - 5 / 7) < 1e-15


@pytest.mark.parametrize("n,k,Dp", [(10, 3, 1_000_000), (40, 39, 5), (7, 1, 4_000_000)])
def test_fig5d_pause(orc, n, k, Dp):
    # Fig. 5d: on time through k, then late by D': 1 - (n-k)D'/(nD' + n(n-1)/(2s))
    P, ttft = 200_000, 1_000_000
    Dl = [ttft + j * P + (Dp if j >= k else 0) for j in range(n)]
    sd, sw, q = orc.qoe_walk(Dl, ttft, P, t=0, m=0, final=True)
    exp = X.qoe_pause(n, k, F(Dp, S), F(S, P))
    assert F(sw - sd, sw) == exp
    assert abs(q - float(exp)) < 1e-15


def test_single_token_cliff(orc):
    # Reading R5: one due token 1 us late -> S_delay = S_whole -> QoE 0
    assert orc.qoe_walk([1_000_001], 1_000_000, 200_000, t=0, m=0, final=True)[2] == 0.0
    assert orc.qoe_walk([1_000_000], 1_000_000, 200_000, t=0, m=0, final=True)[2] == 1.0


# ---------------------------------------------------------------- O2 vs exact-rational walk
def _rand_case(rng):
    # time scale ~ 40 periods so that m stays small for the exact walk
    P = int(rng.choice([1, 3, 200_000, 208_333, 303_030]))
    ttft = int(rng.choice([0, 5, 10 * P, 1_000_000 if P > 3 else 7]))
    span = 40 * P + ttft
    g = int(rng.integers(0, 25))
    D = np.sort(rng.integers(0, span, g)).tolist()
    t = int(rng.integers(max(D) if D else 0, span + 20 * P + 1))
    return P, ttft, D, t


def test_walk_matches_exact_rational(orc):
    rng = np.random.default_rng(7)
    for _ in range(1500):
        P, ttft, D, t = _rand_case(rng)
        speed = F(S, P)
        m_exact = 0 if t < ttft else (t - ttft) // P + 1
        for final in (False, True):
            if final and not D:
                continue
            sd, sw, q = orc.qoe_walk(D, ttft, P, t=t, m=m_exact, final=final)
            esd, esw, eq = X.qoe_exact([F(d, S) for d in D], F(ttft, S), speed, t=F(t, S), final=final)
            assert F(sd, S) == esd and F(sw, S) == esw
            assert abs(q - float(eq)) <= 1e-15
            assert 0.0 <= q <= 1.0
            assert (q == 1.0) == (sd == 0)


def test_sdelay_monotone_in_each_delivery_and_t(orc):
    rng = np.random.default_rng(11)
    for _ in range(400):
        P, ttft, D, t = _rand_case(rng)
        if not D:
            continue
        m = 0 if t < ttft else (t - ttft) // P + 1
        sd0 = orc.qoe_walk(D, ttft, P, t=t, m=m)[0]
        j = int(rng.integers(0, len(D)))
        D2 = list(D)
        D2[j] += int(rng.integers(1, 500_000))
        D2 = D2[:j + 1] + [max(x, D2[j]) for x in D2[j + 1:]]
        D2 = [min(x, t) for x in D2]
        assert orc.qoe_walk(D2, ttft, P, t=t, m=m)[0] >= sd0
        # S_delay(t) nondecreasing in t
        t2 = t + int(rng.integers(1, 3_000_000))
        m2 = 0 if t2 < ttft else (t2 - ttft) // P + 1
        assert orc.qoe_walk(D, ttft, P, t=t2, m=m2)[0] >= sd0


def test_counterexamples_documented(orc):
    # QoE is not monotone in delay: ideal [0,1] s, token 1 at 0.7 s
    q17 = orc.qoe_walk([700_000, 1_700_000], 0, S, 0, 0, final=True)[2]
    q19 = orc.qoe_walk([700_000, 1_900_000], 0, S, 0, 0, final=True)[2]
    assert abs(q17 - 5 / 12) < 1e-15 and abs(q19 - 3 / 7) < 1e-15 and q19 > q17
    # Q_wait(t) is a sawtooth, not monotone (item 3): deliveries [25, 26], TTFT 6, period 2
    a = orc.qoe_walk([25 * S, 26 * S], 6 * S, 2 * S, t=26 * S, m=11)
    b = orc.qoe_walk([25 * S, 26 * S], 6 * S, 2 * S, t=27 * S, m=11)
    assert (a[0], a[1]) == (109 * S, 110 * S) and (b[0], b[1]) == (119 * S, 121 * S)
    assert b[2] > a[2]


def test_qoe_eval_final_and_inflight(orc):
    snap = W.random_small(3, n=9)
    q, sd, sw, m = orc.qoe_eval(snap, snap.now_us)
    for i in range(snap.n):
        D = snap.tl_pool[int(snap.tl_base[i]):int(snap.tl_base[i]) + int(snap.n_deliv[i])]
        t = snap.now_us - int(snap.arrival_us[i])
        P, ttft = int(snap.period_us[i]), int(snap.ttft_us[i])
        mm = min(0 if t < ttft else (t - ttft) // P + 1, int(snap.max_total[i]))
        esd, esw, eq = X.qoe_exact([F(int(d), S) for d in D], F(ttft, S), F(S, P), t=F(t, S), m=mm)
        assert F(int(sd[i]), S) == esd and F(int(sw[i]), S) == esw and m[i] == mm


# ---------------------------------------------------------------- O3-O5 gains
def test_negative_gain_example(orc):
    # P 1 s, ttft 0, d1 0.7 s, now 1.0 s, dt 0.9 s, tau 0.1 s:
    # Q_serve = 5/12, Q_wait = 3/7, gain = -1/84
    snap = _snap_from([dict(arrival_us=0, deliveries_us=[700_000], ctx_len=3, rank=0, running=1)],
                      ttft=0, P=S, now=S)
    gain, key, qw = orc.gain_estimate(snap, S, 900_000, [100_000], [1])
    assert abs(qw[0] - 3 / 7) < 1e-15
    assert abs(gain[0, 0] - (5 / 12 - 3 / 7)) < 1e-15 and gain[0, 0] < 0
    assert key[0, 0] == np.float32((5 / 12 - 3 / 7) / 3)


def test_fig6_serve_shape(orc):
    # Fig. 6: an on-time request keeps perfect QoE when served at a tau that keeps
    # pace (B = 10, 30) and loses it when tau(B) exceeds its period (B = 50); Q_wait is B-free.
    P = 208_333
    ttft = 1_000_000
    D = [ttft + j * P for j in range(20)]
    now = D[-1] + 1
    snap = _snap_from([dict(arrival_us=0, deliveries_us=D, ctx_len=100, rank=0, running=1)],
                      ttft=ttft, P=P, now=now)
    tau = W.tau_table(64, base_us=20_000, per_B_us=3_800)  # tau(50) = 210 ms > P >= tau(30)
    gain, key, qw = orc.gain_estimate(snap, now, 2_000_000, tau, [10, 30, 50])
    qs = qw[0] + gain[:, 0]
    assert abs(qs[0] - 1) < 1e-12 and abs(qs[1] - 1) < 1e-12 and qs[2] < 1 - 1e-6
    assert qw[0] < 1


def test_gain_zero_when_nothing_due_beyond_delivered(orc):
    # g >= m: serving adds no due token, so Q_serve = Q_wait and gain is exactly 0
    snap = W.random_small(5, n=10)
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us,
                                      np.arange(1, snap.tau_us.size + 1))
    t = snap.now_us + snap.horizon_us - snap.arrival_us
    for i in range(snap.n):
        P, ttft = int(snap.period_us[i]), int(snap.ttft_us[i])
        m = min(0 if t[i] < ttft else (int(t[i]) - ttft) // P + 1, int(snap.max_total[i]))
        if snap.n_deliv[i] >= m:
            assert np.all(gain[:, i] == 0.0) and np.all(key[:, i] == 0.0)
    assert np.all(np.signbit(key[key == 0]) == False)  # noqa: E712  (-0 canonicalised)


def test_serve_sdelay_nondecreasing_in_tau(orc):
    # S_delay under serving is nondecreasing in tau(B).  Checked via
    # the exact walk on the oracle's own hypothetical deliveries.
    rng = np.random.default_rng(5)
    for _ in range(200):
        P, ttft, D, t0 = _rand_case(rng)
        now = t0
        dt = int(rng.integers(1, 30 * P + 2))
        t = now + dt
        m = 0 if t < ttft else (t - ttft) // P + 1
        prev = None
        for tau in sorted(rng.integers(1, 3 * P + 2, 6)):
            Dn = D + [now + k * int(tau) for k in range(1, m - len(D) + 1)]
            sd = orc.qoe_walk(Dn, ttft, P, t=t, m=m)[0]
            if prev is not None:
                assert sd >= prev
            prev = sd


# ---------------------------------------------------------------- knapsack pins
def test_spec_greedy_vs_exact_counterexample():
    # S:L230 garble, corrected: greedy {2,3}=0.75 < exact {1,3}=0.85
    q = [F(50, 100), F(40, 100), F(35, 100)]
    l = [4, 3, 2]
    gv, gx = X.greedy_alg1(q, l, 2, 6)
    bv, bs = X.brute_force(q, l, 2, 6)
    dv, dx = X.dp_algorithm2(q, l, 2, 6)
    assert gv == F(75, 100) and gx == [0, 1, 1]
    assert bv == dv == F(85, 100) and bs == {0, 2} and dx == [1, 0, 1]


def test_spec_greedy_examples():
    # all fit -> all; p=[3,2,1], l=[5,5,5], M=10, B=3 -> top two
    assert X.greedy_alg1([1, 1, 1], [1, 1, 1], 5, 10)[1] == [1, 1, 1]
    assert X.greedy_alg1([15, 10, 5], [5, 5, 5], 3, 10)[1] == [1, 1, 0]
    # Algorithm 1 line `break`: a misfit stops the walk even if later items fit
    assert X.greedy_alg1([100, 50, 1], [1, 10, 1], 3, 5)[1] == [1, 0, 0]


def test_dp_equals_brute_force_and_bounds_greedy():
    rng = np.random.default_rng(3)
    for _ in range(150):
        n = int(rng.integers(1, 8))
        M = int(rng.integers(1, 30))
        l = [int(x) for x in rng.integers(1, 12, n)]
        q = [F(int(x), 97) for x in rng.integers(-20, 100, n)]
        for B in range(1, n + 1):
            dv, dx = X.dp_algorithm2(q, l, B, M)
            bv, bs = X.brute_force(q, l, B, M)
            assert dv == bv
            if dv is not None:
                assert sum(l[i] for i in range(n) if dx[i]) <= M and sum(dx) == B
                assert sum(q[i] for i in range(n) if dx[i]) == dv
            gv, gx = X.greedy_alg1(q, l, B, M)
            assert sum(l[i] for i in range(n) if gx[i]) <= M and sum(gx) <= B
            assert gv <= X.brute_force(q, l, B, M, exact_B=False)[0]
            if sum(gx) == B:
                assert gv <= dv


# ---------------------------------------------------------------- O6-O9 schedule
def _snap_from(reqs, ttft, P, now, horizon=2_000_000, tau=(100_000,), M=10_000, cap=W.UINT32_MAX):
    tl = [np.asarray(r["deliveries_us"], np.uint32) for r in reqs]
    g, base, pool = W._pack(tl)
    n = len(reqs)
    return W.Snapshot(
        arrival_us=np.array([r["arrival_us"] for r in reqs], np.int64),
        ttft_us=np.full(n, ttft, np.uint32), period_us=np.full(n, P, np.uint32),
        ctx_len=np.array([r["ctx_len"] for r in reqs], np.uint32), n_deliv=g,
        max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
        rank=np.array([r["rank"] for r in reqs], np.uint32),
        running=np.array([r["running"] for r in reqs], np.uint8), tl_base=base, tl_pool=pool,
        now_us=now, horizon_us=horizon, tau_us=np.asarray(tau, np.uint32), kv_capacity=M, preempt_cap=cap)


def g1_snapshot(cap=W.UINT32_MAX):
    d = json.load(open(os.path.join(GOLD, "g1_decision.json")))
    inp = d["inputs"]
    reqs = []
    for r in inp["requests"]:
        r = dict(r)
        if isinstance(r["deliveries_us"], str):
            r["deliveries_us"] = [500_000 + 50_000 * k for k in range(40)]
        reqs.append(r)
    snap = _snap_from(reqs, inp["ttft_us"], inp["period_us"], inp["now_us"], inp["horizon_us"],
                      inp["tau_us"], inp["kv_capacity"], cap)
    return snap, d


def _names(idx):
    return ["R%d" % i for i in idx]


def test_golden_g1(orc):
    snap, d = g1_snapshot()
    e = d["expected"]
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, [1, 2, 3, 4])
    for i, s in enumerate(e["q_wait"]):
        assert abs(qw[i] - float(F(s))) < 1e-15
    qs = qw[None, :] + gain
    assert np.all(np.abs(qs.T - np.array(e["q_serve_approx_by_B"])) < 1.5e-6)
    for k, v in e["q_serve_exact"].items():
        r, b = k.split("@")
        i, B = int(r[1:]), int(b)
        assert abs(qs[B - 1, i] - float(F(v))) < 1e-15
    assert key[1].tolist() == [np.float32(x) for x in e["key_at_B2"]]
    dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)
    # G1 lists V(4) although no 4 requests fit in M = 1000 (100+300+500+800 > 1000): under
    # reading R16/O6 B_max = 3, so the oracle evaluates B = 1..3 only; V(4) is
    # checked from the B = 4 gains of the G1 selection {R1, R3}.
    assert dec.B_lo == 1 and dec.B_hi == 3
    assert dec.V[:3].tolist() == e["V_by_B"][:3] and dec.V[3] == orc.INT64_MIN
    sel = {B: [int(x[1:]) for x in e["selected_by_B"][B - 1]] for B in (1, 2, 3, 4)}
    for B in (1, 2, 3, 4):
        assert sum(int(np.rint(gain[B - 1, i] * 2.0 ** 32)) for i in sel[B]) == e["V_by_B"][B - 1]
    assert [int(k) for k in dec.kstar[:3]] == [len(sel[B]) for B in (1, 2, 3)]
    assert dec.B_star == e["B_star"]
    for cap_name, exp in e["cap"].items():
        cap = W.UINT32_MAX if cap_name == "off" else int(cap_name)
        dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity, preempt_cap=cap)
        assert sorted(_names(np.nonzero(dec.serve_mask)[0])) == sorted(exp["final"])
        assert _names(dec.admit) == exp["admits"]
        assert _names(dec.preempt) == exp["preempts"]


def test_bounds_examples(orc):
    # l = [2, 3, 10], M = 6 -> B_max = 2.  l = 10 > M is an invalid input under reading
    # R17 (l_i <= M), so the same shortest-first walk is pinned with M = 10 (2+3 <= 10 < 15)
    # and M = 15 (all three fit).
    reqs = [dict(arrival_us=0, deliveries_us=[], ctx_len=c, rank=i, running=0) for i, c in enumerate([2, 3, 10])]
    snap = _snap_from(reqs, 1_000_000, 200_000, 5_000_000, tau=[1000] * 8, M=10)
    assert orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 10).B_hi == 2
    assert orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 15).B_hi == 3
    with pytest.raises(ValueError):
        orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 6)
    # tau = 20000 + 800 B -> B_min = 235 at P = 208,333 and 353 at P = 303,030
    n = 400
    reqs = [dict(arrival_us=0, deliveries_us=[], ctx_len=1, rank=i, running=0) for i in range(n)]
    for P, exp in ((208_333, 235), (303_030, 353)):
        snap = _snap_from(reqs, 1_000_000, P, 3_000_000, tau=W.tau_table(512), M=10_000)
        dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 10_000, flags=3, B_cap=512)
        assert dec.B_hi == n and dec.B_lo == exp


def test_trigger_examples(orc):
    # S:L246-249 / P:L539-543: occupancy 0.95 -> trigger; 0.5 with 50 ms latency vs a 4.8 tok/s
    # reader -> no trigger; 0.5 with 300 ms -> trigger
    reqs = [dict(arrival_us=0, deliveries_us=[1_000_000], ctx_len=c, rank=i, running=1)
            for i, c in enumerate([50, 45])]
    snap = _snap_from(reqs, 1_000_000, 208_333, 2_000_000, M=100)
    dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 100, flags=0)
    assert dec.status == 0 and dec.flags & 1
    snap.ctx_len[:] = [25, 25]
    dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 100, cur_latency_us=50_000, flags=0)
    assert dec.status == 1 and dec.serve_mask.tolist() == [1, 1]
    dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 100, cur_latency_us=300_000, flags=0)
    assert dec.status == 0
    # exactly 90% is not "exceeds" (reading R15)
    snap.ctx_len[:] = [45, 45]
    assert orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 100, flags=0).status == 1


def _gains(orc, snap, B):
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, [B])
    return gain[0], key[0]


def test_schedule_against_algorithm1_and_brute_force(orc):
    """For each B: the oracle's S_B is Algorithm 1 (exact.greedy_alg1 transcription) on the
    oracle's own keys, feasible, and no better than brute force; V(B) sums llrint(gain 2^32);
    B* is the largest argmax; cap special cases behave as reading R18 states."""
    for seed in range(40):
        snap = W.random_small(seed, B_cap=6)
        flags = 1 | (2 if seed % 3 == 0 else 0)
        dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                           preempt_cap=snap.preempt_cap, flags=flags, B_cap=6)
        n = snap.n
        l = snap.ctx_len.astype(int).tolist()
        M = snap.kv_capacity
        srt = sorted(l)
        kM = max(k for k in range(n + 1) if sum(srt[:k]) <= M)
        assert dec.B_hi == min(6, n, kM)
        best = None
        for B in range(dec.B_lo, dec.B_hi + 1):
            g, k = _gains(orc, snap, B)
            v, x = X.greedy_alg1([F(float(kk)) * l[i] for i, kk in enumerate(k)], l, B, M,
                                 rank=snap.rank.tolist())
            sel = [i for i in range(n) if x[i]]
            assert dec.kstar[B - 1] == len(sel)
            assert dec.V[B - 1] == sum(int(np.rint(g[i] * 2.0 ** 32)) for i in sel)
            bf = X.brute_force([F(float(gg)) for gg in g], l, B, M, exact_B=False)[0]
            assert F(float(sum(g[i] for i in sel))) <= bf + F(1, 10 ** 9)
            if best is None or dec.V[B - 1] >= best[0]:
                best = (dec.V[B - 1], B)
        assert dec.B_star == best[1]
        # cap off or not binding -> final set is S_{B*}; Sum l <= M whenever the running set fit
        if snap.preempt_cap == W.UINT32_MAX:
            assert dec.realized == dec.kstar[dec.B_star - 1]
        if sum(l[i] for i in range(n) if snap.running[i]) <= M:
            assert sum(l[i] for i in range(n) if dec.serve_mask[i]) <= M
        if snap.preempt_cap == 0:
            assert dec.preempt.size == 0 or dec.flags & 4


def test_cap_memory_override(orc):
    # Running set above M with cap 0: memory beats the cap (reading R18 step 5)
    reqs = [dict(arrival_us=0, deliveries_us=[1_000_000], ctx_len=c, rank=i, running=1)
            for i, c in enumerate([60, 50, 40])]
    snap = _snap_from(reqs, 1_000_000, 208_333, 2_000_000, M=100, cap=0)
    dec = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, 100, preempt_cap=0)
    assert dec.flags & 4 and dec.admit.size == 0
    assert sum(int(snap.ctx_len[i]) for i in range(3) if dec.serve_mask[i]) <= 100


def test_lqsf_priority_is_the_raw_gain(orc):
    """LQSF (SPEC lqsf_policy; reading R21): the priority is the raw gain (Eq. 4) instead
    of gain / l (Eq. 6).  On G1 at B = 1 the raw-gain order puts R3 first: its gain is exactly 1
    (Q_serve = 1, Q_wait = 0 by the hand check), so V(1) = 2^32; Eq. 6 keeps R1 (gain 10/11 on
    l = 100 beats 1 on l = 800), V(1) = 3904515724 = llrint(10/11 * 2^32)."""
    snap, d = g1_snapshot()
    andes = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)
    lqsf = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                        flags=orc.ORC_FORCE | orc.ORC_LQSF)
    assert int(andes.V[0]) == 3904515724 == round(10 / 11 * 2 ** 32)
    assert int(lqsf.V[0]) == 2 ** 32
    # every B: the LQSF prefix is Algorithm 1 over the raw-gain order (key desc, rank asc)
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, [1, 2, 3])
    for B in range(1, 4):
        g = gain[B - 1].astype(np.float32).astype(np.float64)
        order = sorted(range(snap.n), key=lambda i: (-g[i], int(snap.rank[i])))
        W_, c, V = 0, 0, 0
        for i in order:
            if W_ + int(snap.ctx_len[i]) <= snap.kv_capacity and c + 1 <= B:
                W_ += int(snap.ctx_len[i])
                c += 1
                V += int(np.rint(gain[B - 1][i] * 2.0 ** 32))
            else:
                break
        assert int(lqsf.V[B - 1]) == V and int(lqsf.kstar[B - 1]) == c


def test_maxmin_objective_on_g1(orc):
    """Max-min objective (Appendix A; reading R22): gain = max(Q_min - Q_wait, 0),
    Q_min = the smallest QoE now.  On G1 every request is perfect now (R0 on time; R1's only due
    token is due exactly at t; R2 ahead; R3 has nothing due), so Q_min = 1 and the gains are
    1 - Q_wait = 11/24, 1, 0, 1 for every B.  Priority gain / l orders R1 (1/100), R0
    (11/24/300), R3 (1/800), R2; M = 1000 admits R1 and R0, R3 breaks the walk."""
    snap, d = g1_snapshot()
    o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                     flags=orc.ORC_FORCE | orc.ORC_MAXMIN)
    two32 = 2 ** 32
    v1 = two32
    v2 = two32 + round(11 / 24 * two32)
    assert [int(x) for x in o.V[:3]] == [v1, v2, v2]
    assert [int(x) for x in o.kstar[:3]] == [1, 2, 2]
    assert o.B_star == 3 and o.k_star == 2  # V ties between B = 2 and 3: the larger B (R13)


def test_perfect_count_objective_on_g1(orc):
    """Perfect-count objective (Appendix A; reading R23): gain =
    [1(Q_serve = 1) - 1(Q_wait = 1)] * 1(Q_now = 1).  On G1 all are perfect now; only R3 is
    perfect if served at B = 1 (Q_serve = 1, G1 table) and not when waiting, so its gain is 1 at
    B = 1 and 0 at B >= 2 (Q_serve(2) = 0.9765625); R2 is perfect either way (gain 0)."""
    snap, d = g1_snapshot()
    o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                     flags=orc.ORC_FORCE | orc.ORC_PERFECT)
    assert int(o.V[0]) == 2 ** 32 and int(o.V[1]) == 0 and int(o.V[2]) == 0
    assert o.B_star == 1 and o.k_star == 1 and list(o.admit) == [3]


def test_objectives_reduce_to_zero_when_all_perfect(orc):
    """SPEC gain_maxmin / gain_perfect_count examples: every request perfect and staying perfect
    (deliveries far ahead) -> every gain 0 under both objectives."""
    snap = W.random_small(3, n=6)
    snap.now_us = 1_000_000
    snap.horizon_us = 1
    snap.ttft_us[:] = 10_000_000  # nothing due yet: Q = 1 now, waiting and serving (R4)
    for f in (orc.ORC_MAXMIN, orc.ORC_PERFECT):
        o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity, flags=orc.ORC_FORCE | f)
        assert all(int(v) in (0, -(1 << 63)) for v in o.V)


def test_refiner_on_g1(orc):
    """Overhead-aware refiner (readings R24-R27) on G1 (B* = 2, admits [R1, R3],
    victims [R2, R0], running R0 and R2).  Pair 1 = R1 alone (800 + 100 <= M): its stall is R1's
    prefill, 100 tokens / rate.  At rate 20 tok/s the stall is 5 s: R0 (on time so far) then has
    31 tokens due at t' = 7 s, 26 undelivered, S_delay = sum_{k=5..30} (6 - 0.2k) = 65 s,
    S_whole = 0.2 * 465 = 93 s, so its QoE drops 1 -> 28/93 (R2 stays perfect: 40 tokens far
    ahead); the loss 65/93 exceeds R1's gain 7/11, the pair is rejected and with it the rest:
    the status quo.  At 40 tok/s (2.5 s) R0 drops by 16.9/30.6 < 7/11: R1 is kept; R3's pair
    preempts R2 and R0 and leaves nobody running (loss 0): the decision is unchanged."""
    snap, d = g1_snapshot()
    base = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)
    assert list(base.admit) == [1, 3] and list(base.preempt) == [2, 0]
    two32 = 2 ** 32
    assert round(65 / 93 * two32) > round(7 / 11 * two32) > round(16.9 / 30.6 * two32)
    slow = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                        flags=orc.ORC_FORCE | orc.ORC_REFINE, prefill_tok_s=20)
    assert slow.flags & orc.ORC_FLAG_REFINED
    assert list(slow.admit) == [] and list(slow.preempt) == []
    assert slow.serve_mask.tolist() == [1, 0, 1, 0] and slow.realized == 2
    fast = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                        flags=orc.ORC_FORCE | orc.ORC_REFINE, prefill_tok_s=40)
    assert list(fast.admit) == [1, 3] and list(fast.preempt) == [2, 0]
    assert fast.serve_mask.tolist() == base.serve_mask.tolist()


def test_refiner_zero_overhead_is_identity(orc):
    """SPEC refine: a zero-overhead profile (no prefill or swap cost) makes every stall 0, so
    the loss is 0 and every positive-gain admission is kept (G1's admits both gain > 0)."""
    snap, d = g1_snapshot()
    base = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)
    z = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                     flags=orc.ORC_FORCE | orc.ORC_REFINE, prefill_tok_s=0)
    assert list(z.admit) == list(base.admit) and list(z.preempt) == list(base.preempt)


def test_threaded_oracle_equals_single_thread(orc):
    """The per-B walks (S3/S4) and the per-request walks (S1, gains) are independent; splitting
    them over threads must leave every output unchanged."""
    snap = W.config2()
    kw = dict(preempt_cap=16)
    o1 = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us[:40], snap.kv_capacity, B_cap=40, **kw)
    for th in (2, 3, 8):
        o = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us[:40], snap.kv_capacity, B_cap=40,
                         threads=th, **kw)
        for f in ("serve_mask", "admit", "preempt", "V", "kstar"):
            np.testing.assert_array_equal(getattr(o, f), getattr(o1, f))
        assert (o.B_star, o.realized, o.B_lo, o.B_hi, o.flags, o.k_star) == \
            (o1.B_star, o1.realized, o1.B_lo, o1.B_hi, o1.flags, o1.k_star)
    q1 = orc.qoe_eval(snap, snap.now_us)
    q8 = orc.qoe_eval(snap, snap.now_us, threads=8)
    for a, b in zip(q1, q8):
        np.testing.assert_array_equal(a, b)
    Bl = np.array([1, 7, 40])
    g1 = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, Bl)
    g8 = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, Bl, threads=5)
    for a, b in zip(g1, g8):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- refiner pins fixed by the paper / SPEC
def test_overhead_model_spec_examples(orc):
    """SPEC preemption_overhead / select_mechanism, the R24 model: recompute =
    (0, one prefill of the context), swap = (l / bandwidth, l / bandwidth), the faster round trip,
    ties to swap ("selects the faster one")."""
    # recompute, context 5000 at 5000 tok/s -> (0, 1.0 s)  (no swapping available)
    assert orc.overhead_us(5000, 0, 5000) == (0, 1_000_000)
    # swap, context 4000 at 20000 tok/s -> (0.2, 0.2) s: recompute at 5000 tok/s would take 0.8 s
    assert orc.overhead_us(5000, 20000, 4000) == (200_000, 200_000)
    # equal totals (recompute 0.4 s = swap 0.2 + 0.2 s) -> swap
    assert orc.overhead_us(10000, 20000, 4000) == (200_000, 200_000)
    # recompute total below swap total -> recompute
    assert orc.overhead_us(20000, 20000, 4000) == (0, 200_000)
    # a queued request's admission is its prefill (nothing to swap in)
    assert orc.overhead_us(5000, 20000, 4000, queued=True) == (0, 800_000)


def fig7_snapshot():
    """The refiner's motivating example (Fig. 7), constructed: ten requests of
    context 100 in M = 700 (one victim frees room for one admit), B = 1..7, tau = 50 ms,
    Delta t = 2 s, ttft 1 s, 5 tok/s.
      R1-R3 running, far ahead of schedule (gain 0; R1 the lowest priority by the rank tie-break);
      R4-R7 running, exactly on schedule with no buffer (gain 9/308 each; a 2 s stall costs each
             exactly that QoE: Q_now = 1 -> Q(now + 2 s) = 1 - 9/308);
      R8-R10 queued for 8 s / 1.5 s / 0.5 s (gains ~0.05 / ~0.62 / 1).
    Recomputation at 50 tok/s: admitting a queued request stalls everyone for 2 s."""
    S = 1_000_000
    now = 20 * S
    tls, arr, run = [], [], []
    for _ in range(3):
        arr.append(now - 10 * S)
        tls.append((S + np.arange(80) * 50_000).astype(np.uint32))
        run.append(1)
    for _ in range(4):
        arr.append(now - 10 * S)
        tls.append((S + np.arange(46) * 200_000).astype(np.uint32))
        run.append(1)
    for x in (8 * S, 3 * S // 2, S // 2):
        arr.append(now - x)
        tls.append(np.zeros(0, np.uint32))
        run.append(0)
    n = 10
    g, base, pool = W._pack(tls)
    return W.Snapshot(arrival_us=np.array(arr, np.int64), ttft_us=np.full(n, S, np.uint32),
                      period_us=np.full(n, 200_000, np.uint32), ctx_len=np.full(n, 100, np.uint32), n_deliv=g,
                      max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=np.array([2, 1, 0, 3, 4, 5, 6, 7, 8, 9], np.uint32), running=np.array(run, np.uint8),
                      tl_base=base, tl_pool=pool, now_us=now, horizon_us=2 * S, tau_us=np.full(7, 50_000, np.uint32),
                      kv_capacity=700)


def test_refiner_fig7_toy(orc):
    """Fig. 7 (SPEC refine example): the priority scheduler admits
    {R8, R9, R10} and preempts {R1, R2, R3}; the refiner keeps (R10, R1) and (R9, R2) because each
    admit's gain exceeds the QoE the ongoing requests lose to the stall, rejects (R8, R3) and
    cancels the rest: it "admits only {R9, R10} and preempts {R1, R2}"."""
    snap = fig7_snapshot()
    gain, key, qw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, [7])
    # hand values: R4-R7 on schedule with 10 tokens due in the horizon -> S_d = 9 s, S_w = 308 s
    for i in range(3, 7):
        assert abs(gain[0, i] - 9 / 308) < 1e-15
    assert gain[0, 9] == 1.0 and list(gain[0, :3]) == [0.0, 0.0, 0.0]
    loss = 4 * round(9 / 308 * 2 ** 32)  # four on-schedule requests each lose 9/308 under a 2 s stall
    assert round(gain[0, 8] * 2 ** 32) > loss > round(gain[0, 7] * 2 ** 32) > 0
    base = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)
    assert base.B_star == 7
    assert (base.admit + 1).tolist() == [10, 9, 8] and (base.preempt + 1).tolist() == [1, 2, 3]
    ref = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                       flags=orc.ORC_FORCE | orc.ORC_REFINE, prefill_tok_s=50)
    assert ref.flags & orc.ORC_FLAG_REFINED
    assert (ref.admit + 1).tolist() == [10, 9] and (ref.preempt + 1).tolist() == [1, 2]
    assert ref.serve_mask.tolist() == [0, 0, 1, 1, 1, 1, 1, 0, 1, 1]
    # cheaper admissions (prefill 200 tok/s: 0.5 s stalls cost far less) keep all three pairs
    cheap = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                         flags=orc.ORC_FORCE | orc.ORC_REFINE, prefill_tok_s=200)
    assert (cheap.admit + 1).tolist() == [10, 9, 8] and (cheap.preempt + 1).tolist() == [1, 2, 3]
