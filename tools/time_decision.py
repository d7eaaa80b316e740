"""Quick A/B timing of the config-3 decision (graph replay, L2 flushed between replays, CUDA
events on the launch stream): median / p10 / p90 us for the Andes decision and its variants,
and the L2-warm back-to-back mean.  Env toggles (ANDES_PDL, ...) apply per process;
ANDES_LIB_PATH selects another build; ONLY=andes,lqsf restricts the variants."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

reps = int(os.environ.get("REPS", "60"))
snap = W.config3()
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
out = ctx.alloc_decision(snap.n, 256)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
variants = [("andes", A.ANDES_FORCE), ("lqsf", A.ANDES_FORCE | A.ANDES_LQSF),
            ("maxmin", A.ANDES_FORCE | A.ANDES_OBJ_MAXMIN), ("perfect", A.ANDES_FORCE | A.ANDES_OBJ_PERFECT),
            ("refine", A.ANDES_FORCE | A.ANDES_REFINE)]
only = os.environ.get("ONLY")
with torch.cuda.stream(s):
    for name, fl in variants:
        if only and name not in only.split(","):
            continue

        def call():
            ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=s,
                         preempt_cap=16, flags=fl)
        for _ in range(3):
            call()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
        for _ in range(5):
            g.replay()
        ms = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            ms.append(a.elapsed_time(b) * 1e3)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
        b.synchronize()
        sc = out.scalars.cpu().numpy().view(np.uint32)
        # (the event timer ticks in ~2 us steps here: the mean resolves finer differences)
        res[name] = (round(statistics.median(ms), 1), round(float(np.mean(ms)), 2), round(float(np.percentile(ms, 10)), 1),
                     round(float(np.percentile(ms, 90)), 1), round(a.elapsed_time(b) * 1e3 / reps, 1), int(sc[0]))
tag = " ".join(f"{k}={os.environ[k]}" for k in ("ANDES_PDL", "ANDES_LIB_PATH") if k in os.environ)
print(f"[{tag or 'default'}] us median/mean/p10/p90/warm B*:", res, flush=True)
