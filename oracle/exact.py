"""oracle.exact -- TEST INFRASTRUCTURE ONLY.

Exact-rational reference pieces used to pin the C oracle (never the product):

* ``qoe_exact``      -- Eq. 1-3 on ``fractions.Fraction`` times in
                        seconds, with the ideal timeline of reading R1 and the
                        consumption recurrence of reading R2, the
                        in-flight clamp of reading R3.
* closed forms       -- the four user-experience cases of Fig. 5
                        and "no tokens arrive -> 0", derived in DESIGN.md.
* ``brute_force``    -- exhaustive subsets for Eq. 5.
* ``dp_algorithm2``  -- Algorithm 2 / Appendix C, line by line.
* ``greedy_alg1``    -- Algorithm 1 on exact priorities.

Pure Python; slow by design; for small inputs only.
"""
from __future__ import annotations

from fractions import Fraction as F
from itertools import combinations


def ideal_times(ttft, speed, n, arrival=F(0)):
    """T_i^Ideal = arrival + ttft + (i-1)/speed (reading R1)."""
    return [F(arrival) + F(ttft) + F(i - 1) / F(speed) for i in range(1, n + 1)]


def actual_consumption(deliveries, ideal, speed):
    """T_1 = max(d_1, I_1); T_i = max(d_i, T_{i-1} + 1/speed) (reading R2)."""
    out = []
    for i, d in enumerate(deliveries):
        if i == 0:
            out.append(max(F(d), ideal[0]))
        else:
            out.append(max(F(d), out[-1] + 1 / F(speed)))
    return out


def qoe_exact(deliveries, ttft, speed, t=None, m=None, final=False):
    """Exact (S_delay, S_whole, QoE) as Fractions.

    final=True: all delivered tokens, no clamp (reading R19).
    Otherwise: first m tokens due by relative time t (m defaults to the number of
    ideal times <= t), actual times clamped at t, undelivered tokens at t (R3).
    """
    deliveries = [F(d) for d in deliveries]
    if final:
        m = len(deliveries)
    elif m is None:
        t = F(t)
        m = 0 if t < F(ttft) else int((t - F(ttft)) * F(speed)) + 1
    if m == 0:
        return F(0), F(0), F(1)
    ideal = ideal_times(ttft, speed, m)
    act = actual_consumption(deliveries[:m], ideal, speed)
    T = []
    for j in range(m):
        if j < len(act):
            T.append(act[j] if final else min(act[j], F(t)))
        else:
            T.append(F(t))
    s_delay = sum(T[j] - ideal[j] for j in range(m))
    s_whole = sum(T[m - 1] - ideal[j] for j in range(m))
    q = F(1) if s_whole == 0 else 1 - s_delay / s_whole
    return s_delay, s_whole, q


# --- closed forms of Fig. 5 (derivations in DESIGN.md, "Oracle pins") -------------------
def qoe_ttft_missed(n, D, s):
    """Fig. 5b: every token late by D, then paced at s. QoE = C/(nD + C), C = n(n-1)/(2s)."""
    C = F(n * (n - 1), 2) / F(s)
    return C / (n * F(D) + C)


def qoe_slow_stream(r, s):
    """Fig. 5c: first token on time, then delivered at rate r < s. QoE = s/(2s - r)."""
    return F(s) / (2 * F(s) - F(r))


def qoe_pause(n, k, Dp, s):
    """Fig. 5d: on time through token k, tokens k+1..n late by D'.
    QoE = 1 - (n-k)D' / (nD' + n(n-1)/(2s))."""
    return 1 - (n - k) * F(Dp) / (n * F(Dp) + F(n * (n - 1), 2) / F(s))


# --- knapsack references -----------------------------------------------------------------
def brute_force(q, l, B, M, exact_B=True):
    """max sum q_i x_i  s.t. sum x = B (or <= B), sum l x <= M  (Eq. 5). Returns (value, set)
    or (None, None) if infeasible."""
    n = len(q)
    best, best_set = None, None
    sizes = [B] if exact_B else range(0, B + 1)
    for k in sizes:
        if k > n:
            continue
        for S in combinations(range(n), k):
            if sum(l[i] for i in S) <= M:
                v = sum(q[i] for i in S)
                if best is None or v > best:
                    best, best_set = v, set(S)
    return best, best_set


def dp_algorithm2(q, l, B, M):
    """Algorithm 2, transcribed line by line (1-based i).
    Returns (Q_max, x) with x a 0/1 list, or (None, None) when dp[N][B][:] is all -inf."""
    NEG = None  # -infinity
    N = len(q)

    def lt(a, b):  # a < b with None = -inf
        if b is None:
            return False
        if a is None:
            return True
        return a < b

    dp = [[[NEG] * (M + 1) for _ in range(B + 1)] for _ in range(N + 1)]
    choice = [[[0] * (M + 1) for _ in range(B + 1)] for _ in range(N + 1)]
    dp[0][0][0] = 0
    for i in range(1, N + 1):
        for b in range(0, min(i, B) + 1):
            for m in range(0, M + 1):
                if lt(dp[i][b][m], dp[i - 1][b][m]):  # request i is not served
                    dp[i][b][m] = dp[i - 1][b][m]
                    choice[i][b][m] = 0
                if b >= 1 and m >= l[i - 1]:
                    prev = dp[i - 1][b - 1][m - l[i - 1]]
                    if prev is not None and lt(dp[i][b][m], prev + q[i - 1]):  # request i is served
                        dp[i][b][m] = prev + q[i - 1]
                        choice[i][b][m] = 1
    row = dp[N][B]
    Q_max = None
    m_cur = None
    for m in range(M + 1):
        if row[m] is not None and (Q_max is None or row[m] > Q_max):
            Q_max, m_cur = row[m], m
    if Q_max is None:
        return None, None
    b_cur = B
    x = [0] * (N + 1)
    for i in range(N, 0, -1):
        x[i] = choice[i][b_cur][m_cur]
        if x[i] == 1:
            m_cur -= l[i - 1]
            b_cur -= 1
    return Q_max, x[1:]


def greedy_alg1(q, l, B, M, rank=None):
    """Algorithm 1 on exact priorities q/l; ties to the smaller rank (R10)."""
    n = len(q)
    rank = list(range(n)) if rank is None else rank
    order = sorted(range(n), key=lambda i: (-F(q[i]) / F(l[i]), rank[i]))
    Mc = Nc = 0
    x = [0] * n
    for i in order:
        if Mc + l[i] <= M and Nc + 1 <= B:
            x[i] = 1
            Mc += l[i]
            Nc += 1
        else:
            break
    return sum(q[i] for i in range(n) if x[i]), x
