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


def test_tracker_graph_iterations(A, orc):
    """The serving iteration captured ONCE into a CUDA graph -- copies of the decision time and of
    the deltas from pinned host memory, andes_tracker_append_dev (count read on the device),
    andes_schedule with now_dev (time read on the device) -- and replayed with a new time and new
    deltas every iteration: every decision equals the oracle's on the host-updated state."""
    snap = dataclasses.replace(W.with_room(W.config2(), 12), preempt_cap=16)
    ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    tau = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()
    out = ctx.alloc_decision(snap.n, int(tau.numel()))
    maxc = 1024
    hnow = torch.zeros(1, dtype=torch.int64).pin_memory()
    hcnt = torch.zeros(1, dtype=torch.int32).pin_memory()
    hidx = torch.zeros(maxc, dtype=torch.int32).pin_memory()
    hts = torch.zeros(maxc, dtype=torch.int64).pin_memory()
    dnow = torch.zeros(1, dtype=torch.int64, device="cuda")
    dcnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    didx = torch.zeros(maxc, dtype=torch.int32, device="cuda")
    dts = torch.zeros(maxc, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()

    def check(cur):
        sc = out.scalars.cpu().numpy().view(np.uint32)
        g = dict(mask=out.serve_mask.cpu().numpy()[:snap.n], admit=out.admit.cpu().numpy().view(np.uint32)[:sc[2]],
                 preempt=out.preempt.cpu().numpy().view(np.uint32)[:sc[3]], sc=sc, V=out.V.cpu().numpy(),
                 kstar=out.kstar.cpu().numpy().view(np.uint32))
        o = orc.schedule(cur, cur.now_us, cur.horizon_us, cur.tau_us, cur.kv_capacity, preempt_cap=cur.preempt_cap)
        assert_decision_equal(g, o)
        return o

    with torch.cuda.stream(s):
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out, stream=s,
                     preempt_cap=snap.preempt_cap)
    s.synchronize()
    cur = snap
    o = check(cur)
    g = None
    for it in range(6):
        served = np.nonzero(o.serve_mask)[0]
        assert served.size <= maxc
        t_abs = cur.now_us + int(cur.tau_us[max(o.B_star, 1) - 1])
        hnow[0] = t_abs
        hcnt[0] = served.size
        hidx[:served.size] = torch.from_numpy(served.astype(np.int32))
        hts[:served.size] = t_abs
        with torch.cuda.stream(s):
            if g is None:  # captured at the first iteration, replayed at every later one
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    dnow.copy_(hnow, non_blocking=True)
                    dcnt.copy_(hcnt, non_blocking=True)
                    didx.copy_(hidx, non_blocking=True)
                    dts.copy_(hts, non_blocking=True)
                    ctx.tracker_append_dev(req, snap.n, didx, dts, dcnt, serve_mask=out.serve_mask, stream=s)
                    ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, out=out,
                                 stream=s, preempt_cap=snap.preempt_cap, now_dev=dnow)
            g.replay()
        s.synchronize()
        cur = dataclasses.replace(_host_append(cur, served, t_abs), now_us=t_abs)
        np.testing.assert_array_equal(req["n_deliv"].cpu().numpy().view(np.uint32), cur.n_deliv)
        o = check(cur)


@pytest.mark.parametrize("flags", ["andes", "lqsf", "maxmin", "perfect", "refine", "debug"])
def test_schedule_now_dev_equals_host_now(A, flags):
    """andes_schedule with the time read on the device (now_dev) equals the host-time call, at
    several times and under every flavour (the objectives' second scan and the refiner included)."""
    snap = W.config2()
    fl = A.ANDES_FORCE | {"andes": 0, "lqsf": A.ANDES_LQSF, "maxmin": A.ANDES_OBJ_MAXMIN,
                          "perfect": A.ANDES_OBJ_PERFECT, "refine": A.ANDES_REFINE,
                          "debug": A.ANDES_DEBUG_CHECKS}[flags]
    ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    tau = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()
    for dt in (0, 150_000, 2_500_000):
        now = snap.now_us + dt
        a = ctx.schedule(req, snap.n, now, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16, flags=fl)
        dnow = torch.tensor([now], dtype=torch.int64, device="cuda")
        b = ctx.schedule(req, snap.n, snap.now_us - 777_777, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16,
                         flags=fl, now_dev=dnow)
        torch.cuda.synchronize()
        for f in ("scalars", "V", "kstar", "serve_mask", "admit", "preempt"):
            x, y = getattr(a, f), getattr(b, f)
            if f == "admit":
                k = int(a.scalars[2])
                x, y = x[:k], y[:k]
            if f == "preempt":
                k = int(a.scalars[3])
                x, y = x[:k], y[:k]
            assert torch.equal(x, y), (flags, dt, f)


def test_tracker_dev_count_above_max_is_rejected(A):
    snap = W.with_room(W.random_small(5, n=8, max_tokens=10), 4)
    ctx = A.Context(max_requests=snap.n, max_B=16, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    before = req["n_deliv"].cpu().numpy().copy()
    idx = torch.arange(4, dtype=torch.int32, device="cuda")
    ts = torch.full((4,), int(snap.now_us), dtype=torch.int64, device="cuda")
    cnt = torch.tensor([5], dtype=torch.int32, device="cuda")  # > the 4 slots
    ctx.tracker_append_dev(req, snap.n, idx, ts, cnt)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(req["n_deliv"].cpu().numpy(), before)
    with pytest.raises(RuntimeError, match="CAPACITY|capacity"):
        ctx.tracker_append_dev(req, snap.n, idx, ts, cnt)
    cnt.fill_(2)
    ctx.tracker_append_dev(req, snap.n, idx, ts, cnt)
    torch.cuda.synchronize()
    after = req["n_deliv"].cpu().numpy()
    np.testing.assert_array_equal(after[:2], before[:2] + 1)
    np.testing.assert_array_equal(after[2:], before[2:])


def test_decision_export_zero_copy(A):
    """AndesDecision.export_host: the decision's head written into mapped pinned memory equals the
    device outputs, and the exported next batch is exactly the serve mask (realized entries)."""
    snap = dataclasses.replace(W.config2(), preempt_cap=16)
    ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
    req = A.requests_to(snap)
    tau = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()
    pmax, smax = 512, 1024
    buf = torch.zeros(A.decision_export_bytes(256, pmax, smax), dtype=torch.uint8).pin_memory()
    hnow = torch.tensor([snap.now_us + 40_000], dtype=torch.int64).pin_memory()
    for flags in (A.ANDES_FORCE, A.ANDES_FORCE | A.ANDES_REFINE, 0):
        out = ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16,
                           flags=flags, export_host=buf, export_preempt=pmax, export_served=smax, now_dev=hnow)
        torch.cuda.synchronize()
        sc, V, adm, pre, srv = A.decision_export_views(buf, 256, pmax, smax)
        done = A.decision_export_done(buf, 256, pmax, smax)
        assert int(done[0]) == 1
        done[0] = 0
        dsc = out.scalars.cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(sc, dsc)
        np.testing.assert_array_equal(V, out.V.cpu().numpy())
        np.testing.assert_array_equal(adm[:dsc[2]], out.admit.cpu().numpy()[:dsc[2]])
        np.testing.assert_array_equal(pre[:min(dsc[3], pmax)], out.preempt.cpu().numpy()[:min(dsc[3], pmax)])
        mask = out.serve_mask.cpu().numpy()[:snap.n]
        assert int(dsc[1]) == int(mask.sum())
        np.testing.assert_array_equal(np.sort(srv[:dsc[1]]), np.nonzero(mask)[0])
