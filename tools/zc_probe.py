import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2404_16283_b200 as A, workloads as W
snap = W.config3(); sn = W.with_room(snap, 60); n = sn.n
ctx = A.Context(max_requests=n, max_B=256, max_tokens=sn.n_tokens + 64)
req = A.requests_to(sn); tau = torch.from_numpy(sn.tau_us.view(np.int32)).cuda()
out = ctx.alloc_decision(n, 256); s = torch.cuda.Stream()
hnow = torch.tensor([sn.now_us], dtype=torch.int64).pin_memory()
dnow = hnow.cuda()
hcnt = torch.tensor([170], dtype=torch.int32).pin_memory(); dcnt = hcnt.cuda()
hidx = torch.arange(1024, dtype=torch.int32).pin_memory(); didx = hidx.cuda()
hts = torch.full((1024,), sn.now_us, dtype=torch.int64).pin_memory(); dts = hts.cuda()
hexp = torch.zeros(A.decision_export_bytes(256, 4096), dtype=torch.uint8).pin_memory()
def T(name, f, reps=20):
    with torch.cuda.stream(s):
        for _ in range(3): f()
        s.synchronize()
        ms = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); f(); b.record(s); b.synchronize(); ms.append(a.elapsed_time(b) * 1e3)
    print(f"{name:28s} {np.median(ms):8.1f} us", flush=True)
kw = dict(preempt_cap=16, flags=A.ANDES_FORCE, stream=s)
T("schedule host now", lambda: ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, **kw))
T("schedule now_dev device", lambda: ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=dnow, **kw))
T("schedule now_dev pinned", lambda: ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, now_dev=hnow, **kw))
T("schedule + export", lambda: ctx.schedule(req, n, sn.now_us, sn.horizon_us, tau, sn.kv_capacity, out=out, export_host=hexp, export_preempt=4096, **kw))
T("tracker dev inputs", lambda: ctx.tracker_append_dev(req, n, didx, dts, dcnt, stream=s), reps=5)
T("tracker pinned inputs", lambda: ctx.tracker_append_dev(req, n, hidx, hts, hcnt, stream=s), reps=5)
T("copy 12KB H2D", lambda: didx.copy_(hidx, non_blocking=True))
