"""workloads -- seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no QoE, gain, priority,
knapsack or bound computation): it only draws request populations, delivery
timestamps and the synthetic latency table, following the recipe in DESIGN.md
("Input recipe"), which restates SURVEY.md section 8(d):

* lengths: lognormal fits to Table 2, clamped;
* TTFT target max(input/5000, 1) s; speeds 4.8 / 3.3 tok/s;
* arrivals: cyclic burst, intensity 2, duration 35%, or Poisson;
* latency table tau(B) = 20000 + 800 B microseconds -- synthetic ("OPT-13B-like"
  in BASELINE.json has no PAPER.md counterpart; labelled synthetic);
* KV capacity M = 163,840 tokens; Delta t = 2 s.

All times are integer microseconds; delivery timestamps are microseconds since
the request's arrival (u32), packed per request in request order.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

UINT32_MAX = 0xFFFFFFFF

# Table 2 lognormal fits: (input mu, sigma, output mu, sigma)
LENGTH_FITS = {
    "sharegpt": (7.0696, 1.4087, 5.7160, 0.6888),
    "arxiv": (9.6191, 0.5848, 6.3742, 0.2490),
    "coding": (5.5955, 1.3559, 7.1993, 1.6728),
}
READ_PERIOD_US = 208_333    # 4.8 tok/s, round(1e6/4.8)
LISTEN_PERIOD_US = 303_030  # 3.3 tok/s, round(1e6/3.3)
KV_CAPACITY = 163_840
HORIZON_US = 2_000_000
B_CAP = 256


def tau_table(B_cap: int = B_CAP, base_us: int = 20_000, per_B_us: int = 800) -> np.ndarray:
    """Synthetic decode latency tau(B) = base + per_B * B (microseconds), index B-1."""
    B = np.arange(1, B_cap + 1, dtype=np.int64)
    return (base_us + per_B_us * B).astype(np.uint32)


@dataclass
class Snapshot:
    """SoA request table + decision parameters (the C-ABI's AndesRequests/AndesSchedParams)."""
    arrival_us: np.ndarray
    ttft_us: np.ndarray
    period_us: np.ndarray
    ctx_len: np.ndarray
    n_deliv: np.ndarray
    max_total: np.ndarray
    start_off_us: np.ndarray
    rank: np.ndarray
    running: np.ndarray
    tl_base: np.ndarray
    tl_pool: np.ndarray
    now_us: int = 0
    horizon_us: int = HORIZON_US
    tau_us: np.ndarray = field(default_factory=tau_table)
    kv_capacity: int = KV_CAPACITY
    preempt_cap: int = UINT32_MAX
    cur_latency_us: int = 0
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.arrival_us.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.tl_pool.shape[0])

    def subset(self, idx, align: int = 4) -> "Snapshot":
        """Requests idx (re-packed pool), same parameters."""
        idx = np.asarray(idx, dtype=np.int64)
        parts = [self.tl_pool[int(self.tl_base[i]):int(self.tl_base[i]) + int(self.n_deliv[i])] for i in idx]
        g, base, pool = _pack(parts, align)
        return replace(self, arrival_us=self.arrival_us[idx].copy(), ttft_us=self.ttft_us[idx].copy(),
                       period_us=self.period_us[idx].copy(), ctx_len=self.ctx_len[idx].copy(),
                       n_deliv=g.copy(), max_total=self.max_total[idx].copy(),
                       start_off_us=self.start_off_us[idx].copy(), rank=self.rank[idx].copy(),
                       running=self.running[idx].copy(), tl_base=base, tl_pool=pool)


POOL_ALIGN = 4  # tokens: every timeline starts on a 16-byte boundary (the scan's aligned fast path)


def _pack(timelines, align: int = POOL_ALIGN):
    """Pack per-request timelines into one pool, request order; each timeline starts at a
    multiple of `align` tokens (padding repeats the previous value; it is never a valid token)."""
    g = np.array([len(t) for t in timelines], dtype=np.uint32)
    span = ((g.astype(np.uint64) + np.uint64(align - 1)) // np.uint64(align)) * np.uint64(align)
    base = np.zeros(len(timelines), np.uint64)
    if len(timelines):
        base[1:] = np.cumsum(span[:-1])
    total = int(span.sum())
    pool = np.zeros(total, np.uint32)
    for i, t in enumerate(timelines):
        if len(t):
            b = int(base[i])
            pool[b:b + len(t)] = np.asarray(t, np.uint32)
            pool[b + len(t):b + int(span[i])] = pool[b + len(t) - 1]
    return g, base, pool


def with_room(snap: Snapshot, extra: int, align: int = POOL_ALIGN) -> Snapshot:
    """The same snapshot with `extra` free token slots after every timeline (a device-resident
    tracker appends into them, andes_tracker_append); timelines stay `align`-aligned."""
    g = snap.n_deliv.astype(np.int64)
    span = (g + extra + align - 1) // align * align
    base = np.zeros(snap.n, np.int64)
    if snap.n:
        base[1:] = np.cumsum(span[:-1])
    pool = np.zeros(int(span.sum()) if snap.n else 0, np.uint32)
    src = snap.tl_base.astype(np.int64)
    for i in range(snap.n):
        if g[i]:
            pool[base[i]:base[i] + g[i]] = snap.tl_pool[src[i]:src[i] + g[i]]
    return replace(snap, tl_base=base.astype(np.uint64), tl_pool=pool)


def sample_lengths(rng, n, dataset="sharegpt", in_clamp=(1, 32768), out_clamp=(1, 8192)):
    mi, si, mo, so = LENGTH_FITS[dataset]
    inp = np.clip(np.rint(rng.lognormal(mi, si, n)), *in_clamp).astype(np.int64)
    out = np.clip(np.rint(rng.lognormal(mo, so, n)), *out_clamp).astype(np.int64)
    return inp, out


def cyclic_burst_arrivals(rng, n, mean_rate_per_s, cycle_s=1200.0, burst_frac=0.35, intensity=2.0):
    """Cyclic burst: each cycle a burst phase at intensity x mean for
    burst_frac of the cycle, then a base phase whose rate keeps the cycle mean.
    Returns n arrival times (seconds, ascending) from t=0."""
    r_b = intensity * mean_rate_per_s
    r_0 = (1.0 - intensity * burst_frac) / (1.0 - burst_frac) * mean_rate_per_s
    out = []
    t = 0.0
    while len(out) < n:
        phase = (t % cycle_s) / cycle_s
        rate = r_b if phase < burst_frac else r_0
        t += rng.exponential(1.0 / rate)
        out.append(t)
    return np.array(out[:n])


def snapshot(n, seed=1, dataset="sharegpt", listen_frac=0.0, window_s=1200.0, arrivals="burst",
             tau_gap_B=B_CAP, kv_capacity=KV_CAPACITY, preempt_cap=UINT32_MAX, B_cap=B_CAP,
             horizon_us=HORIZON_US, name="") -> Snapshot:
    """Live-population snapshot at `now` (recipe: DESIGN.md "Input recipe").

    Classes: 30% running/recently served (g ~ U[1, out-1]); 40% preempted mid-stream
    (same, with one pause U[0.5, 5] s at a uniform index); 30% queued (g = 0).
    First token at a + Exp(2 s) + input/5000 s; later tokens spaced tau(tau_gap_B)
    +-10% jitter; everything truncated at `now`. Running flag: class-0 requests in
    arrival order while their context lengths fit in M.
    """
    rng = np.random.default_rng(seed)
    tau = tau_table(B_cap)
    inp, out = sample_lengths(rng, n, dataset)
    if arrivals == "burst":
        arr_s = cyclic_burst_arrivals(rng, n, n / window_s)
    else:  # Poisson
        arr_s = np.cumsum(rng.exponential(window_s / n, n))
    now_s = float(arr_s[-1]) + 0.05
    arr_us = np.rint(arr_s * 1e6).astype(np.int64)
    now_us = int(np.rint(now_s * 1e6))
    age_us = now_us - arr_us
    cls = rng.choice(3, size=n, p=[0.3, 0.4, 0.3])
    ttft = np.maximum(200 * inp, 1_000_000).astype(np.uint32)          # max(len/5000, 1) s
    period = np.where(rng.random(n) < listen_frac, LISTEN_PERIOD_US, READ_PERIOD_US).astype(np.uint32)
    gap = float(tau[min(tau_gap_B, B_cap) - 1])
    timelines = []
    for i in range(n):
        if cls[i] == 2 or out[i] <= 1:
            timelines.append(np.zeros(0, np.uint32))
            continue
        g = int(rng.integers(1, out[i]))
        first = rng.exponential(2e6) + inp[i] * 200.0
        gaps = gap * (1.0 + rng.uniform(-0.1, 0.1, g - 1))
        ts = first + np.concatenate([[0.0], np.cumsum(gaps)])
        if cls[i] == 1 and g > 1:
            k = int(rng.integers(1, g))
            ts[k:] += rng.uniform(0.5e6, 5e6)
        ts = np.floor(ts)
        ts = ts[ts <= age_us[i]]
        timelines.append(ts.astype(np.uint32))
    g, base, pool = _pack(timelines)
    ctx = (inp + g).astype(np.uint32)
    running = np.zeros(n, np.uint8)
    W = 0
    for i in range(n):
        if cls[i] == 0 and g[i] > 0 and W + int(ctx[i]) <= kv_capacity:
            running[i] = 1
            W += int(ctx[i])
    return Snapshot(arrival_us=arr_us, ttft_us=ttft, period_us=period, ctx_len=ctx, n_deliv=g,
                    max_total=np.full(n, UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                    rank=np.arange(n, dtype=np.uint32), running=running, tl_base=base, tl_pool=pool,
                    now_us=now_us, horizon_us=horizon_us, tau_us=tau, kv_capacity=kv_capacity,
                    preempt_cap=preempt_cap, name=name or f"{dataset}-{n}-s{seed}")


def config1_population(seed=1):
    """BASELINE config 1: 8 requests, prompts U[150, 600], outputs U[20, 120],
    arrivals U[0, 2] s, in arrival order.  Returns (prompt, out_len, arrival_us)."""
    rng = np.random.default_rng(seed)
    n = 8
    prompt = rng.integers(150, 601, n)
    out_len = rng.integers(20, 121, n)
    arr = rng.integers(0, 2_000_001, n).astype(np.int64)
    order = np.argsort(arr, kind="stable")
    return prompt[order], out_len[order], arr[order]


def config1(seed=1) -> Snapshot:
    """The first decision of the config-1 driver: every request arrived, no token delivered yet;
    ttft 1 s, 4.8 tok/s, M = 2048, tau(B) for B = 1..8, Delta t = 2 s, cap off."""
    prompt, out_len, arr = config1_population(seed)
    n = prompt.size
    g, base, pool = _pack([np.zeros(0, np.uint32)] * n)
    return Snapshot(arrival_us=arr, ttft_us=np.full(n, 1_000_000, np.uint32), period_us=np.full(n, READ_PERIOD_US, np.uint32),
                    ctx_len=prompt.astype(np.uint32), n_deliv=g, max_total=np.full(n, UINT32_MAX, np.uint32),
                    start_off_us=np.zeros(n, np.uint32), rank=np.arange(n, dtype=np.uint32),
                    running=np.zeros(n, np.uint8), tl_base=base, tl_pool=pool, now_us=int(arr.max()),
                    horizon_us=HORIZON_US, tau_us=tau_table(8), kv_capacity=2048, name="config1")


def config2(seed=1) -> Snapshot:
    """BASELINE config 2: 4K ShareGPT-shaped snapshot, all readers, B=1..256, P_cap off."""
    return snapshot(4096, seed=seed, listen_frac=0.0, window_s=300.0, name=f"cfg2-4k-s{seed}")


def config3(seed=1, n=65536) -> Snapshot:
    """BASELINE config 3: burst at 2x capacity, 64K live, 50/50 reading/listening, P_cap = 16."""
    return snapshot(n, seed=seed, listen_frac=0.5, window_s=1200.0, preempt_cap=16,
                    name=f"cfg3-{n // 1024}k-s{seed}")


def tile(snap: Snapshot, reps: int, running_copies: int | None = None) -> Snapshot:
    """reps copies of a snapshot back to back (same shape and statistics), ranks renumbered
    0..n*reps-1; the running flag is kept in the first `running_copies` copies only (default all)."""
    n, T = snap.n, snap.n_tokens
    base = np.concatenate([snap.tl_base + np.uint64(k * T) for k in range(reps)])
    run = np.tile(snap.running, reps)
    if running_copies is not None:
        run[running_copies * n:] = 0
    return replace(snap, arrival_us=np.tile(snap.arrival_us, reps), ttft_us=np.tile(snap.ttft_us, reps),
                   period_us=np.tile(snap.period_us, reps), ctx_len=np.tile(snap.ctx_len, reps),
                   n_deliv=np.tile(snap.n_deliv, reps), max_total=np.tile(snap.max_total, reps),
                   start_off_us=np.tile(snap.start_off_us, reps),
                   rank=np.arange(n * reps, dtype=np.uint32), running=run, tl_base=base,
                   tl_pool=np.tile(snap.tl_pool, reps), name=f"{snap.name}x{reps}")


def shard(snap: Snapshot, lo: int, hi: int) -> Snapshot:
    """Requests lo..hi-1 as a contiguous shard with its own pool (the multi-GPU layout)."""
    b0 = int(snap.tl_base[lo]) if lo < snap.n else snap.n_tokens
    b1 = int(snap.tl_base[hi - 1]) + int(snap.n_deliv[hi - 1]) if hi > lo else b0
    sl = slice(lo, hi)
    return replace(snap, arrival_us=snap.arrival_us[sl], ttft_us=snap.ttft_us[sl], period_us=snap.period_us[sl],
                   ctx_len=snap.ctx_len[sl], n_deliv=snap.n_deliv[sl], max_total=snap.max_total[sl],
                   start_off_us=snap.start_off_us[sl], rank=snap.rank[sl], running=snap.running[sl],
                   tl_base=(snap.tl_base[sl] - np.uint64(b0)).astype(np.uint64),
                   tl_pool=snap.tl_pool[b0:b1], name=f"{snap.name}[{lo}:{hi}]")


def config4(seed=1, reps=16) -> Snapshot:
    """BASELINE config 4: 2^20 live requests (config 3 scaled: 16 copies of the 64K snapshot,
    the running batch kept in the first copy so it fits M), for the sharded decision."""
    return tile(config3(seed), reps, running_copies=1)


SWEEP_RHOS = tuple(round(0.50 + 0.05 * k, 2) for k in range(32))  # load factors 0.50 .. 2.05


def sweep_scenario(seed: int, rho: float, n_base: int = 2000, window_s: float = 1200.0, listen_frac: float = 0.5,
                   dataset: str = "sharegpt"):
    """One config-5 scenario: a 20-minute cyclic-burst trace of ~n_base*rho requests
    whose timelines are COMPLETE (g = output length), drawn from a parametric load model instead of
    a scheduler: queue wait ~ Exp(2 s * rho^3), prefill input/5000 s, token gaps
    tau(min(256, ceil(128 rho))) +-10%, one pause U[0.5, 5] s with probability min(0.5, 0.1 rho^2).
    Vectorised (no per-request Python loop).  Returns the SoA arrays (relative timestamps, us)."""
    rng = np.random.default_rng([int(seed), int(round(rho * 100))])
    n = max(1, int(round(n_base * rho)))
    inp, out = sample_lengths(rng, n, dataset)
    g = out.astype(np.int64)  # completed requests deliver their whole output
    # arrivals: unit-rate Poisson mapped through the cyclic-burst cumulative intensity
    mean_rate = n / window_s
    r_b, burst = 2.0 * mean_rate, 0.35
    r_0 = (1.0 - 2.0 * burst) / (1.0 - burst) * mean_rate
    lam_cycle = window_s * (burst * r_b + (1 - burst) * r_0)
    u = np.cumsum(rng.exponential(1.0, n))
    cyc, rem = np.divmod(u, lam_cycle)
    tb = burst * window_s * r_b
    t_in = np.where(rem < tb, rem / r_b, burst * window_s + (rem - tb) / r_0)
    arr_us = np.rint((cyc * window_s + t_in) * 1e6).astype(np.int64)
    wait = rng.exponential(2e6 * rho ** 3, n)
    first = wait + 200.0 * inp
    gap = float(tau_table(B_CAP)[min(256, int(np.ceil(128 * rho))) - 1])
    T = int(g.sum())
    start = np.concatenate([[0], np.cumsum(g)[:-1]])
    steps = gap * (1.0 + rng.uniform(-0.1, 0.1, T))
    steps[start] = first
    pause_on = (rng.random(n) < min(0.5, 0.1 * rho * rho)) & (g > 1)
    k = np.minimum(rng.integers(1, np.maximum(g, 2)), np.maximum(g - 1, 1))
    plen = rng.uniform(0.5e6, 5e6, n)
    steps[start[pause_on] + k[pause_on]] += plen[pause_on]
    ts = np.cumsum(steps)
    seg0 = np.repeat(ts[start] - steps[start], g)
    pool = np.floor(ts - seg0).astype(np.uint32)
    ttft = np.maximum(200 * inp, 1_000_000).astype(np.uint32)
    period = np.where(rng.random(n) < listen_frac, LISTEN_PERIOD_US, READ_PERIOD_US).astype(np.uint32)
    return dict(arrival_us=arr_us, ttft_us=ttft, period_us=period, ctx_len=(inp + g).astype(np.uint32),
                n_deliv=g.astype(np.uint32), tl_pool=pool)


def sweep(scenarios, n_base: int = 2000) -> tuple[Snapshot, np.ndarray]:
    """Concatenation of sweep_scenario(seed, rho) for every (seed, rho) in `scenarios` (requests
    grouped by scenario, pools packed back to back, ranks unique); returns the population and the
    request offsets u32[S+1] of the scenarios (BASELINE config 5: 32 seeds x SWEEP_RHOS)."""
    parts = [sweep_scenario(sd, rho, n_base) for sd, rho in scenarios]
    cat = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    g = cat["n_deliv"].astype(np.int64)
    span = (g + POOL_ALIGN - 1) // POOL_ALIGN * POOL_ALIGN  # 16-byte aligned timelines
    base = np.concatenate([[0], np.cumsum(span)[:-1]]).astype(np.int64)
    src = np.concatenate([[0], np.cumsum(g)[:-1]])
    pool = np.zeros(int(span.sum()), np.uint32)
    pool[np.repeat(base - src, g) + np.arange(int(g.sum()))] = cat["tl_pool"]
    cat["tl_pool"] = pool
    base = base.astype(np.uint64)
    n = int(g.size)
    off = np.concatenate([[0], np.cumsum([p["n_deliv"].size for p in parts])]).astype(np.uint32)
    snap = Snapshot(arrival_us=cat["arrival_us"], ttft_us=cat["ttft_us"], period_us=cat["period_us"],
                    ctx_len=cat["ctx_len"], n_deliv=cat["n_deliv"], max_total=np.full(n, UINT32_MAX, np.uint32),
                    start_off_us=np.zeros(n, np.uint32), rank=np.arange(n, dtype=np.uint32),
                    running=np.zeros(n, np.uint8), tl_base=base, tl_pool=cat["tl_pool"], now_us=0,
                    name=f"sweep-{len(parts)}")
    return snap, off


def sim_trace(seed: int, rho: float, window_s: float = 120.0, rate_at_rho1: float = 2.0, listen_frac: float = 0.5,
              dataset: str = "sharegpt", max_prompt: int = 32768, max_out: int = 8192) -> dict:
    """A request trace for the serving-loop simulator (NEXT-3, andes_simulate): cyclic-burst
    arrivals (intensity 2, 35% burst; the cycle shortened to the window) at
    rho * rate_at_rho1 requests/s on average (rate_at_rho1 ~ the synthetic tau(B) model's service
    rate at M = 163,840 for ShareGPT-shaped requests), Table-2 lengths (clamped), TTFT target
    max(input/5000, 1) s, reading / listening speeds.  Timelines get room for the
    whole output (16-byte aligned starts).  Arrival order = rank."""
    rng = np.random.default_rng([int(seed), int(round(rho * 100)), 7])
    n = max(1, int(round(rate_at_rho1 * rho * window_s)))
    inp, out = sample_lengths(rng, n, dataset, in_clamp=(1, max_prompt), out_clamp=(1, max_out))
    arr_s = cyclic_burst_arrivals(rng, n, n / window_s, cycle_s=window_s)
    arr = np.rint(arr_s * 1e6).astype(np.int64)
    span = (out.astype(np.int64) + POOL_ALIGN - 1) // POOL_ALIGN * POOL_ALIGN
    base = np.concatenate([[0], np.cumsum(span)[:-1]]).astype(np.uint64)
    return dict(n=n, arrival_us=arr, ttft_us=np.maximum(200 * inp, 1_000_000).astype(np.uint32),
                period_us=np.where(rng.random(n) < listen_frac, LISTEN_PERIOD_US, READ_PERIOD_US).astype(np.uint32),
                prompt_len=inp.astype(np.uint32), output_len=out.astype(np.uint32), tl_base=base,
                tl_len=int(span.sum()), name=f"sim-s{seed}-rho{rho:.2f}")


def config5_scenarios(seeds: int = 32, rhos=SWEEP_RHOS):
    """BASELINE config 5: 1024 scenarios = 32 trace seeds x 32 load factors."""
    return [(sd, rho) for sd in range(1, seeds + 1) for rho in rhos]


def random_small(seed, n=None, max_tokens=40, B_cap=16, edge=True, align: int = POOL_ALIGN) -> Snapshot:
    """Small adversarial instances for parity: arbitrary periods, ttft, offsets,
    max_total caps, deliveries ahead of / behind schedule, pauses, ties."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 12)) if n is None else n
    now = int(rng.integers(2_000_000, 20_000_000))
    arr = now - rng.integers(0, 15_000_000, n)
    # periods >= 50 ms keep m (tokens due by now + dt) below ~500 for the literal walk
    period = rng.choice([50_000, 100_000, 208_333, 303_030, 999_983], n).astype(np.uint32)
    ttft = rng.choice([0, 1, 500_000, 1_000_000, 1_300_000, 3_000_000], n).astype(np.uint32)
    timelines = []
    for i in range(n):
        g = int(rng.integers(0, max_tokens + 1)) if rng.random() < 0.8 else 0
        if g == 0:
            timelines.append(np.zeros(0, np.uint32))
            continue
        age = int(now - arr[i])
        ts = np.sort(rng.integers(0, max(age, 1) + 1, g))
        if edge and rng.random() < 0.3:
            ts = np.minimum(ts, ttft[i] + np.arange(g) * int(period[i]))  # on/ahead of schedule
            ts = np.sort(np.minimum(ts, age))
        timelines.append(ts.astype(np.uint32))
    g, base, pool = _pack(timelines, align)
    ctx = rng.integers(1, 60, n).astype(np.uint32)
    mt = np.where(rng.random(n) < 0.2, g + rng.integers(0, 5, n), UINT32_MAX).astype(np.uint32)
    off = np.where(rng.random(n) < 0.3, rng.integers(0, 3_000_000, n), 0).astype(np.uint32)
    rank = rng.permutation(n).astype(np.uint32)
    running = (rng.random(n) < 0.5).astype(np.uint8)
    tau = np.sort(rng.integers(1, 400_000, B_cap)).astype(np.uint32)
    horizon = int(rng.choice([1, 250_000, 2_000_000, 5_000_000]))
    M = int(max(int(ctx.max()), int(rng.integers(20, 300))))
    return Snapshot(arrival_us=arr.astype(np.int64), ttft_us=ttft, period_us=period, ctx_len=ctx, n_deliv=g,
                    max_total=mt, start_off_us=off, rank=rank, running=running, tl_base=base, tl_pool=pool,
                    now_us=now, horizon_us=horizon, tau_us=tau, kv_capacity=M,
                    preempt_cap=int(rng.choice([UINT32_MAX, 0, 1, 2])), name=f"rand-s{seed}")


def long_requests(seed, n=200, lo=5_000, hi=30_000, align: int = POOL_ALIGN) -> Snapshot:
    """Long-output requests (5K-30K tokens each): nearly every tile's head request started more
    than 4096 tokens earlier, so the scan's carry comes by look-back (or its direct fallback).
    Deliveries follow the ideal schedule with jitter, stalls that make them late, and catch-ups;
    a few requests are empty or tiny so that short segments sit between the long ones."""
    rng = np.random.default_rng(seed)
    P = rng.choice([20_000, 33_333, 50_000], n).astype(np.uint32)
    ttft = rng.choice([0, 300_000, 1_000_000], n).astype(np.uint32)
    timelines = []
    span = 0
    for i in range(n):
        g = int(rng.integers(lo, hi + 1)) if rng.random() < 0.9 else int(rng.integers(0, 3))
        j = np.arange(g, dtype=np.int64)
        d = int(ttft[i]) + j * int(P[i]) + rng.integers(-int(P[i]) // 2, int(P[i]) // 2 + 1, g)
        for _ in range(int(rng.integers(0, 4))):  # stalls: every later token shifted
            if g:
                d[int(rng.integers(0, g)):] += int(rng.integers(0, 40)) * int(P[i])
        d = np.maximum.accumulate(np.maximum(d, 0))
        timelines.append(d.astype(np.uint32))
        span = max(span, int(d[-1]) if g else 0)
    g, base, pool = _pack(timelines, align)
    now = span + 1_000_000
    return Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=ttft, period_us=P,
                    ctx_len=rng.integers(1, 4096, n).astype(np.uint32), n_deliv=g,
                    max_total=np.full(n, UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                    rank=rng.permutation(n).astype(np.uint32), running=(rng.random(n) < 0.5).astype(np.uint8),
                    tl_base=base, tl_pool=pool, now_us=now, horizon_us=2_000_000, tau_us=tau_table(),
                    kv_capacity=1 << 20, preempt_cap=UINT32_MAX, name=f"long-s{seed}")
