"""Where bench.py's e2e serving iteration goes (its loop as it stands: tracker update on pinned
inputs, decision with now_dev, zero-copy export polled by the host): per step the host staging,
the graph.replay() call, the wait for the export's completion word, and the device span of the
replay from CUDA events around it (median over the steps)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

steps = int(os.environ.get("STEPS", "40"))
snap = W.config3()
sn = W.with_room(snap, steps + 8)
n = sn.n
ctx = A.Context(max_requests=n, max_B=256, max_tokens=sn.n_tokens + 64)
req = A.requests_to(sn)
tau = torch.from_numpy(sn.tau_us.view(np.int32)).cuda()
out = ctx.alloc_decision(n, 256)
stream = torch.cuda.Stream()
maxc, pmax = min(n, 1024), min(n, 4096)
hnow = torch.zeros(1, dtype=torch.int64).pin_memory()
hts = torch.zeros(maxc, dtype=torch.int64).pin_memory()
hexp = torch.zeros(A.decision_export_bytes(256, pmax, maxc), dtype=torch.uint8).pin_memory()
np_sc, _, np_adm, np_pre, np_srv = A.decision_export_views(hexp, 256, pmax, maxc)
o_srv = 32 + 12 * 256 + 4 * pmax
srv_t = hexp[o_srv:o_srv + 4 * maxc].view(torch.int32)
np_done = A.decision_export_done(hexp, 256, pmax, maxc)
cnt_t = hexp[4:8].view(torch.int32)
np_now, np_ts = hnow.numpy(), hts.numpy()
kw = dict(preempt_cap=sn.preempt_cap, flags=A.ANDES_FORCE, stream=stream, export_host=hexp, export_preempt=pmax,
          export_served=maxc)
only = os.environ.get("ONLY", "")


kw_noexp = dict(preempt_cap=sn.preempt_cap, flags=A.ANDES_FORCE, stream=stream)


def iteration():
    # ONLY: decision (no tracker update), tracker (the update alone), noexport (tracker + decision
    # without the zero-copy export), nonow (as noexport, the time passed by value)
    if only != "decision":
        ctx.tracker_append_dev(req, n, srv_t, hts, cnt_t, serve_mask=out.serve_mask, stream=stream)
    if only == "tracker":
        return
    if only == "noexport":
        ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=hnow, **kw_noexp)
    elif only == "nonow":
        ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, **kw_noexp)
    else:
        ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=hnow, **kw)


now = sn.now_us
res = {"host": [], "replay": [], "wait": [], "device": [], "wall": []}
with torch.cuda.stream(stream):
    ctx.schedule(req, n, now, sn.horizon_us, tau, sn.kv_capacity, out=out, **kw)
    stream.synchronize()
    graph = None
    for k in range(steps + 3):
        t0 = time.perf_counter()
        cnt = int(np_sc[1])
        now += int(sn.tau_us[max(int(np_sc[0]), 1) - 1])
        np_now[0] = now
        np_ts[:cnt] = now
        np_done[0] = 0
        if graph is None:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                iteration()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t1 = time.perf_counter()
        a.record(stream)
        graph.replay()
        b.record(stream)
        t2 = time.perf_counter()
        while np_done[0] == 0 and only not in ("tracker", "noexport", "nonow"):
            pass
        t3 = time.perf_counter()
        b.synchronize()
        if k >= 3:
            res["host"].append(t1 - t0)
            res["replay"].append(t2 - t1)
            res["wait"].append(t3 - t2)
            res["wall"].append(t3 - t0)
            res["device"].append(a.elapsed_time(b) * 1e-3)
print(f"[e2e split{(' ' + only) if only else ''}] " + ", ".join(f"{k} {1e6 * float(np.median(v)):.1f} us" for k, v in res.items()))
