"""BASELINE config 1 driver (SURVEY 8(d) per-config inputs): 8 requests, ttft 1 s, 4.8 tok/s,
prompts U[150, 600], outputs U[20, 120], arrivals U[0, 2] s, M = 2048, tau(B) = 20 ms + 0.8 ms B,
Delta t = 2 s, preemption cap off; 200 iterations in zero-overhead mode: the clock advances by
tau(realized), every served request receives one token, finished requests leave.

Shared by the CPU decision-quality test (oracle + brute force + exact DP) and the GPU parity
test (GPU == oracle on every iteration, Algorithm 2 on the GPU); holds no method arithmetic:
`decide(snap)` returns the oracle's decision, `on_iter(snap, decision)` checks it."""
from __future__ import annotations

import numpy as np

import workloads as W


def run(decide, iters=200, seed=1, on_iter=None):
    prompt, out_len, arr = W.config1_population(seed)
    n = prompt.size
    tau = W.tau_table(8)
    now = int(arr.max())
    toks = [[] for _ in range(n)]
    running = np.zeros(n, np.uint8)
    alive = np.ones(n, bool)
    decided = 0
    for it in range(iters):
        idx = np.nonzero(alive & (arr <= now))[0]
        if idx.size == 0:
            now += 100_000
            continue
        g, base, pool = W._pack([np.asarray(toks[i], np.uint32) for i in idx])
        snap = W.Snapshot(arrival_us=arr[idx], ttft_us=np.full(idx.size, 1_000_000, np.uint32),
                          period_us=np.full(idx.size, 208_333, np.uint32),
                          ctx_len=(prompt[idx] + g).astype(np.uint32), n_deliv=g,
                          max_total=np.full(idx.size, W.UINT32_MAX, np.uint32),
                          start_off_us=np.zeros(idx.size, np.uint32), rank=idx.astype(np.uint32),
                          running=running[idx], tl_base=base, tl_pool=pool, now_us=now, horizon_us=2_000_000,
                          tau_us=tau, kv_capacity=2048, name=f"config1-it{it}")
        od = decide(snap)
        decided += 1
        if on_iter is not None:
            on_iter(snap, od)
        served = idx[np.nonzero(od.serve_mask)[0]]
        realized = max(1, served.size)
        now += int(tau[min(realized, tau.size) - 1])
        running[:] = 0
        for i in served:
            toks[i].append(now - int(arr[i]))
            running[i] = 1
            if len(toks[i]) >= out_len[i]:
                alive[i] = False
                running[i] = 0
    return decided


class QualityTracker:
    """Greedy (Algorithm 1) vs exact (Eq. 5) on every iteration, in the objective's
    exact integer units (llrint(gain 2^32), reading R9): for every candidate B, the brute-force
    optimum over subsets of size <= B (and exactly B) that fit M bounds V(B) from above; the
    ratio V(B*) / max_B OPT(B) is the decision's quality (the paper's greedy-vs-3D-DP comparison,
    P:L1072-1075)."""

    def __init__(self, orc, exact_dp=None):
        self.orc = orc
        self.exact_dp = exact_dp  # optional callable(q, l, B, M) -> (best, Vb) (Algorithm 2)
        self.ratios = []
        self.checked_B = 0
        self.gaps = 0

    def __call__(self, snap, od):
        from oracle import exact as X
        if od.status != 0 or od.B_star == 0:
            return
        Bs = list(range(od.B_lo, od.B_hi + 1))
        gain, key, qw = self.orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, Bs)
        l = [int(x) for x in snap.ctx_len]
        M = int(snap.kv_capacity)
        best_any = None
        for b, B in enumerate(Bs):
            q = [int(v) for v in np.rint(gain[b] * 2.0 ** 32).astype(np.int64)]
            le, _ = X.brute_force(q, l, B, M, exact_B=False)
            eq, _ = X.brute_force(q, l, B, M, exact_B=True)
            assert le is not None and int(od.V[B - 1]) <= le, (snap.name, B, int(od.V[B - 1]), le)
            if eq is not None and int(od.kstar[B - 1]) == B:
                assert int(od.V[B - 1]) <= eq
            if self.exact_dp is not None:
                best, Vb = self.exact_dp(q, l, B, M)
                assert best == eq, (snap.name, B, best, eq)  # Algorithm 2 == brute force (|S| = B)
                assert max(v for v in Vb if v is not None) == le  # best over every size <= B
            self.checked_B += 1
            if int(od.V[B - 1]) < le:
                self.gaps += 1
            best_any = le if best_any is None else max(best_any, le)
        vstar = int(od.V[od.B_star - 1])
        assert vstar <= best_any
        if best_any > 0:
            self.ratios.append(vstar / best_any)

    def summary(self):
        r = np.asarray(self.ratios) if self.ratios else np.ones(1)
        return {"iterations_with_positive_optimum": len(self.ratios), "B_values_checked": self.checked_B,
                "B_values_with_greedy_below_exact": self.gaps, "ratio_min": float(r.min()),
                "ratio_mean": float(r.mean()), "ratio_p10": float(np.percentile(r, 10))}
