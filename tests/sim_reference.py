"""TEST INFRASTRUCTURE: the serving loop of andes_simulate (include/andes.h, NEXT-3) on the host
with the CPU oracle's decision in the loop -- the same rules written out plainly: live = arrived
(a_i <= now) and unfinished (g_i < out_i), rank = trace index, running = served in the previous
iteration, l = prompt + g, max_total unknown (UINT32_MAX); every served request receives one token
at now' = now + tau(min(max(realized, 1), B_cap)); no live request -> the clock jumps to the next
arrival.  Returns (n_deliv, timelines, iterations)."""
from __future__ import annotations

import numpy as np

import workloads as W


def simulate_reference(orc, tr, tau, kv_capacity, horizon_us=2_000_000, preempt_cap=W.UINT32_MAX, flags=1,
                       max_iters=0):
    n = tr["n"]
    arr, out = tr["arrival_us"], tr["output_len"]
    g = np.zeros(n, np.int64)
    served = np.zeros(n, np.uint8)
    tls = [[] for _ in range(n)]
    now = int(arr[0])
    it = 0
    B_cap = int(tau.size)
    while True:
        hi = int(np.searchsorted(arr, now, side="right"))
        idx = np.array([i for i in range(hi) if g[i] < out[i]], np.int64)
        if hi == n and idx.size == 0:
            break
        if max_iters and it >= max_iters:
            break
        if idx.size == 0:
            now = int(arr[hi])
            continue
        gg, base, pool = W._pack([np.asarray(tls[i], np.uint32) for i in idx])
        snap = W.Snapshot(arrival_us=arr[idx].copy(), ttft_us=tr["ttft_us"][idx].copy(),
                          period_us=tr["period_us"][idx].copy(), ctx_len=(tr["prompt_len"][idx] + gg).astype(np.uint32),
                          n_deliv=gg, max_total=np.full(idx.size, W.UINT32_MAX, np.uint32),
                          start_off_us=np.zeros(idx.size, np.uint32), rank=idx.astype(np.uint32),
                          running=served[idx].copy(), tl_base=base, tl_pool=pool, now_us=now, horizon_us=horizon_us,
                          tau_us=tau, kv_capacity=kv_capacity)
        o = orc.schedule(snap, now, horizon_us, tau, kv_capacity, preempt_cap=preempt_cap, flags=flags | orc.ORC_FORCE)
        realized = max(1, min(o.realized, B_cap))
        t_new = now + int(tau[realized - 1])
        for k, i in enumerate(idx):
            served[i] = o.serve_mask[k]
            if o.serve_mask[k]:
                tls[i].append(t_new - int(arr[i]))
                g[i] += 1
        now = t_new
        it += 1
    return g, tls, it
