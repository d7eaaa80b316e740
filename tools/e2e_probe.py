"""Where the e2e serving iteration's wall time goes (bench.py e2e_incremental's loop): host staging
+ served-set update, graph.replay() call, synchronize, and the device time of the replay (events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

snap = W.config3()
sn = W.with_room(snap, 60)
n = sn.n
ctx = A.Context(max_requests=n, max_B=256, max_tokens=sn.n_tokens + 64)
req = A.requests_to(sn)
tau = torch.from_numpy(sn.tau_us.view(np.int32)).cuda()
out = ctx.alloc_decision(n, 256)
s = torch.cuda.Stream()
maxc, pmax = 1024, 4096
hnow = torch.zeros(1, dtype=torch.int64).pin_memory()
hcnt = torch.zeros(1, dtype=torch.int32).pin_memory()
hidx = torch.zeros(maxc, dtype=torch.int32).pin_memory()
hts = torch.zeros(maxc, dtype=torch.int64).pin_memory()
hsc = torch.empty(8, dtype=torch.int32).pin_memory()
hV = torch.empty(256, dtype=torch.int64).pin_memory()
hadm = torch.empty(256, dtype=torch.int32).pin_memory()
hpre = torch.empty(pmax, dtype=torch.int32).pin_memory()
dnow = torch.zeros(1, dtype=torch.int64, device="cuda")
dcnt = torch.zeros(1, dtype=torch.int32, device="cuda")
didx = torch.zeros(maxc, dtype=torch.int32, device="cuda")
dts = torch.zeros(maxc, dtype=torch.int64, device="cuda")
variant = os.environ.get("V", "full")


hst = torch.zeros(16 + 12 * maxc, dtype=torch.uint8).pin_memory()
dst = torch.zeros(16 + 12 * maxc, dtype=torch.uint8, device="cuda")
pk = ctx.alloc_decision(n, 256, packed=True)
head = pk.packed_offsets[4] + 4 * pmax
hout = torch.empty(head, dtype=torch.uint8).pin_memory()


def iteration():
    if variant == "full":
        dnow.copy_(hnow, non_blocking=True)
        dcnt.copy_(hcnt, non_blocking=True)
        didx.copy_(hidx, non_blocking=True)
        dts.copy_(hts, non_blocking=True)
    if variant == "packed":
        dst.copy_(hst, non_blocking=True)
    if variant == "notracker":
        ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=dnow, stream=s,
                     preempt_cap=sn.preempt_cap, flags=A.ANDES_FORCE)
        return
    ctx.tracker_append_dev(req, n, didx, dts, dcnt, serve_mask=out.serve_mask, stream=s)
    ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=dnow, stream=s,
                 preempt_cap=sn.preempt_cap, flags=A.ANDES_FORCE)
    if variant == "packed":
        hout.copy_(pk.packed[:head], non_blocking=True)
    if variant == "full":
        hsc.copy_(out.scalars, non_blocking=True)
        hV.copy_(out.V, non_blocking=True)
        hadm.copy_(out.admit, non_blocking=True)
        hpre.copy_(out.preempt[:pmax], non_blocking=True)


hnow[0] = sn.now_us
with torch.cuda.stream(s):
    ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, stream=s, preempt_cap=16)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        iteration()
    for _ in range(5):
        g.replay()
    s.synchronize()
    tr, ts_, dev = [], [], []
    for k in range(30):
        hnow[0] = sn.now_us + 1000 * k
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(s)
        g.replay()
        b.record(s)
        t1 = time.perf_counter()
        s.synchronize()
        t2 = time.perf_counter()
        tr.append(t1 - t0)
        ts_.append(t2 - t1)
        dev.append(a.elapsed_time(b) * 1e-3)
served = np.nonzero(sn.running)[0].astype(np.int32)
th = []
for k in range(30):
    t0 = time.perf_counter()
    sc = hsc.numpy().view(np.uint32)
    na, npre = int(sc[2]), int(sc[3])
    sv = np.union1d(np.setdiff1d(served, hpre.numpy()[:npre], assume_unique=True), hadm.numpy()[:na])
    hidx.numpy()[:sv.size] = sv
    hts.numpy()[:sv.size] = 5
    th.append(time.perf_counter() - t0)
md = lambda x: 1e6 * float(np.median(x))  # noqa: E731
print(f"[{variant}] replay call {md(tr):.1f} us, sync {md(ts_):.1f} us, device {md(dev):.1f} us, host update {md(th):.1f} us")
