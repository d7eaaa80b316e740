"""Small decisions and QoE evaluations for compute-sanitizer (memcheck / racecheck runs): every
decision flavour, debug checks, the sharded steps at world 1, the tracker update (host count and
device count with pinned inputs), the decision with now_dev and the zero-copy export, the
peer-memory all-gather at world 1, the serving-loop simulator and the fused cooperative kernel
(ANDES_FUSED=1 when set in the environment)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

ctx = A.Context(max_requests=8192, max_B=64, max_tokens=1 << 22, max_running=4096)
for seed in range(6):
    snap = W.random_small(seed, align=[4, 1][seed % 2], n=30, max_tokens=300, B_cap=16)
    req = A.requests_to(snap)
    tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
    for fl in (1, 1 | 16, 1 | 32, 1 | 64, 1 | 128):
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=2, flags=fl)
    ctx.qoe_eval(req, snap.n, snap.now_us, A.ANDES_EVAL_FINAL)
    ctx.qoe_eval(req, snap.n, snap.now_us + snap.horizon_us, A.ANDES_EVAL_INFLIGHT)
    ctx.qoe_eval(req, snap.n, snap.now_us, A.ANDES_EVAL_INFLIGHT, outputs=("q",))
    ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=2,
                 flags=1 | A.ANDES_DEBUG_CHECKS)
    # sharded entry point, world 1 (the exchange is a device copy)
    sh = ctx.shard_init(1, 0, int(tau.numel()))
    out = ctx.alloc_shard_decision(snap.n, int(tau.numel()))
    A.schedule_sharded(ctx, sh, req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity,
                       lambda a, b: b.copy_(a), out=out, preempt_cap=2)
    # tracker update with room
    sr = W.with_room(snap, 4)
    rq2 = A.requests_to(sr)
    d = ctx.schedule(rq2, sr.n, sr.now_us, sr.horizon_us, tau, sr.kv_capacity)
    idx = torch.nonzero(d.serve_mask[:sr.n]).flatten().to(torch.int32)
    ts = torch.full((idx.numel(),), sr.now_us + 1000, dtype=torch.int64, device="cuda")
    ctx.tracker_append(rq2, sr.n, idx if idx.numel() else None, ts if idx.numel() else None, serve_mask=d.serve_mask)
    # round 2: the replayable serving step -- the tracker update reading pinned host inputs with
    # the count on the device, the decision time from pinned memory, the zero-copy export
    hts = torch.full((64,), sr.now_us + 2000, dtype=torch.int64).pin_memory()
    hexp = torch.zeros(A.decision_export_bytes(int(tau.numel()), 64, 64), dtype=torch.uint8).pin_memory()
    hnow = torch.tensor([sr.now_us + 2000], dtype=torch.int64).pin_memory()
    d = ctx.schedule(rq2, sr.n, sr.now_us, sr.horizon_us, tau, sr.kv_capacity, preempt_cap=2, export_host=hexp,
                     export_preempt=64, export_served=64, now_dev=hnow)
    torch.cuda.synchronize()
    srv = hexp[hexp.numel() - 4 * 64:].view(torch.int32)
    cnt = hexp[4:8].view(torch.int32)
    ctx.tracker_append_dev(rq2, sr.n, srv, hts, cnt, serve_mask=d.serve_mask)
# the peer-memory all-gather at world 1 (arena slot copies, flag publish and wait)
cm = A.Comm(1, 0, 4096)
cm.connect([cm.handle])
src = torch.arange(1000, dtype=torch.int32, device="cuda")
dstb = torch.zeros(1000, dtype=torch.int32, device="cuda")
for _ in range(3):
    cm.allgather(src, dstb)
torch.cuda.synchronize()
assert torch.equal(src, dstb)
cm.close()
snap = W.long_requests(3, n=60, lo=5000, hi=9000)
req = A.requests_to(snap)
ctx.qoe_eval(req, snap.n, snap.now_us, A.ANDES_EVAL_INFLIGHT)
tr = W.sim_trace(2, 1.5, window_s=8.0, rate_at_rho1=2.5, max_prompt=3000, max_out=30)
sc = A.Context(max_requests=tr["n"], max_B=16, max_tokens=tr["tl_len"] + 64)
sc.simulate(tr, torch.from_numpy(W.tau_table(16).view(np.int32)).cuda(), 12_000, flags=16)
torch.cuda.synchronize()
print("sanitize run ok")
