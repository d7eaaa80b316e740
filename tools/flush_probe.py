"""Decision graph timing under different L2 / host-sync regimes (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

snap = W.config3()
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
s = torch.cuda.Stream()
out = ctx.alloc_decision(snap.n, 256)
with torch.cuda.stream(s):
    for _ in range(3):
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16, out=out, stream=s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16, out=out, stream=s)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    N = 30

    def run(mode):
        ts = []
        for k in range(N):
            if mode in ("flush", "flush_sync"):
                flush.zero_()
            if mode == "flush_sync":
                s.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            if mode != "warm":
                b.synchronize()
            ts.append((a, b))
        torch.cuda.synchronize()
        return np.median([a.elapsed_time(b) for a, b in ts]) * 1e3

    for mode in ("warm", "flush", "flush_sync", "warm"):
        print(os.environ.get("ANDES_PDL", "0"), mode, round(run(mode), 1), "us")
