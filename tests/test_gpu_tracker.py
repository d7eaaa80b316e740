"""andes_tracker_append (-m gpu): the device-resident Request Tracker update between decisions
(P:L337).  Several serving iterations of config-2-shaped state: decision on the GPU, the served
requests each receive one token at now + tau(B*) appended on the device; the device arrays must
equal the same update done on the host with numpy, and every decision must equal the oracle's
on the host-updated snapshot."""
import dataclasses

import numpy as np
import pytest

import workloads as W
from conftest import assert_decision_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


def _host_append(snap, served, t_abs):
    pool = snap.tl_pool.copy()
    g = snap.n_deliv.copy()
    l = snap.ctx_len.copy()
    for i in served:
        pool[int(snap.tl_base[i]) + int(g[i])] = np.uint32(t_abs - int(snap.arrival_us[i]))
        g[i] += 1
        l[i] += 1
    running = np.zeros(snap.n, np.uint8)
    running[served] = 1
    return dataclasses.replace(snap, tl_pool=pool, n_deliv=g, ctx_len=l, running=running)


@pytest.mark.parametrize("name", ["config2", "random"])
def test_tracker_iterations_match_host_and_oracle(A, orc, name):
    snap = W.config2() if name == "config2" else W.random_small(17, n=200, max_tokens=60, B_cap=16)
    snap = dataclasses.replace(W.with_room(snap, 12), preempt_cap=16 if name == "config2" else snap.preempt_cap)
    ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    tau = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()
    out = ctx.alloc_decision(snap.n, int(tau.numel()))
    now = snap.now_us
    for it in range(8):
        cur = dataclasses.replace(snap, now_us=now)
        ctx.schedule(req, snap.n, now, snap.horizon_us, tau, snap.kv_capacity, out=out,
                     preempt_cap=cur.preempt_cap)
        torch.cuda.synchronize()
        sc = out.scalars.cpu().numpy().view(np.uint32)
        g = dict(mask=out.serve_mask.cpu().numpy()[:snap.n], admit=out.admit.cpu().numpy().view(np.uint32)[:sc[2]],
                 preempt=out.preempt.cpu().numpy().view(np.uint32)[:sc[3]], sc=sc, V=out.V.cpu().numpy(),
                 kstar=out.kstar.cpu().numpy().view(np.uint32))
        o = orc.schedule(cur, now, cur.horizon_us, cur.tau_us, cur.kv_capacity, preempt_cap=cur.preempt_cap)
        assert_decision_equal(g, o)
        served = np.nonzero(o.serve_mask)[0]
        Bs = max(o.B_star, 1)
        t_abs = now + int(cur.tau_us[Bs - 1])
        idx = torch.from_numpy(served.astype(np.int32)).cuda()
        ts = torch.full((served.size,), t_abs, dtype=torch.int64, device="cuda")
        ctx.tracker_append(req, snap.n, idx, ts, serve_mask=out.serve_mask)
        torch.cuda.synchronize()
        snap = _host_append(cur, served, t_abs)
        np.testing.assert_array_equal(req["n_deliv"].cpu().numpy().view(np.uint32), snap.n_deliv)
        np.testing.assert_array_equal(req["ctx_len"].cpu().numpy().view(np.uint32), snap.ctx_len)
        np.testing.assert_array_equal(req["running"].cpu().numpy(), snap.running)
        gp = req["tl_pool"].cpu().numpy().view(np.uint32)
        for i in served:
            b = int(snap.tl_base[i])
            np.testing.assert_array_equal(gp[b:b + int(snap.n_deliv[i])], snap.tl_pool[b:b + int(snap.n_deliv[i])])
        now = t_abs


def test_tracker_rejects_a_full_timeline(A):
    snap = W.random_small(3, n=6, max_tokens=8)
    snap = W.with_room(snap, 0, align=1)  # no room at all
    ctx = A.Context(max_requests=64, max_B=16, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    i = 0 if snap.n > 1 else 0
    idx = torch.tensor([i], dtype=torch.int32, device="cuda")
    ts = torch.tensor([snap.now_us], dtype=torch.int64, device="cuda")
    ctx.tracker_append(req, snap.n, idx, ts)
    torch.cuda.synchronize()
    assert int(req["n_deliv"][i].item()) == int(snap.n_deliv[i])  # dropped
    with pytest.raises(A.AndesError) as ei:
        ctx.tracker_append(req, snap.n, None, None)
    assert ei.value.rc == A.ANDES_E_CAPACITY
