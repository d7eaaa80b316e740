"""Error paths of the C ABI (-m gpu; include/andes.h "Conventions"): capacity overflows are
always reported (ANDES_F_TRUNCATED on the failing decision, ANDES_E_CAPACITY on the next call);
ANDES_DEBUG_CHECKS data preconditions (timestamps, ranks, context lengths) report
ANDES_E_RANGE on the next call and never fire on valid inputs; the _host entry point rejects
NULL required arrays before copying anything."""
import dataclasses

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


@pytest.fixture(scope="module")
def ctx(A):
    return A.Context(max_requests=1 << 14, max_B=256, max_tokens=1 << 22)


def _tau(snap):
    return torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()


def _sched(A, ctx, snap, flags=1):
    d = ctx.schedule(A.requests_to(snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), snap.kv_capacity,
                     preempt_cap=snap.preempt_cap, flags=flags)
    torch.cuda.synchronize()
    return d


def _expect_next_call_fails(A, ctx, rc):
    ok = W.random_small(1, n=5)
    with pytest.raises(A.AndesError) as ei:
        _sched(A, ctx, ok)
    assert ei.value.rc == rc, str(ei.value)
    _sched(A, ctx, ok)  # the error word was cleared by the failing call


def test_running_set_above_capacity(A, ctx):
    n = 5000  # > 4096 running requests
    tl = [np.zeros(0, np.uint32)] * n
    g, base, pool = W._pack(tl)
    snap = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                      period_us=np.full(n, 208_333, np.uint32), ctx_len=np.ones(n, np.uint32), n_deliv=g,
                      max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                      rank=np.arange(n, dtype=np.uint32), running=np.ones(n, np.uint8), tl_base=base,
                      tl_pool=pool, now_us=5_000_000, horizon_us=2_000_000, tau_us=W.tau_table(8),
                      kv_capacity=1_000_000)
    d = _sched(A, ctx, snap)
    assert d.scalar("flags") & A.ANDES_F_TRUNCATED
    _expect_next_call_fails(A, ctx, A.ANDES_E_CAPACITY)


def test_debug_checks_silent_on_valid_inputs(A, ctx, orc):
    for snap in (W.config2(), W.random_small(7, n=30), W.random_small(8, n=30, align=1)):
        d = _sched(A, ctx, snap, flags=1 | A.ANDES_DEBUG_CHECKS)
        assert not d.scalar("flags") & A.ANDES_F_TRUNCATED
        _sched(A, ctx, W.random_small(1, n=5))  # no pending error


def _bad(kind):
    snap = W.random_small(3, n=20, max_tokens=30)
    snap = dataclasses.replace(snap, tl_pool=snap.tl_pool.copy(), rank=snap.rank.copy(), ctx_len=snap.ctx_len.copy())
    i = int(np.argmax(snap.n_deliv))
    b = int(snap.tl_base[i])
    if kind == "decreasing":
        snap.tl_pool[b] = snap.tl_pool[b + 1] + 1  # d_1 > d_2
    elif kind == "future":
        snap.tl_pool[b + int(snap.n_deliv[i]) - 1] = np.uint32(int(snap.now_us - snap.arrival_us[i]) + 1)
    elif kind == "rank":
        snap.rank[5] = snap.rank[11]
    elif kind == "ctx":
        snap.ctx_len[2] = snap.kv_capacity + 1
    return snap


@pytest.mark.parametrize("kind", ["decreasing", "future", "rank", "ctx"])
def test_debug_checks_report_range(A, ctx, kind):
    snap = _bad(kind)
    assert snap.n_deliv.max() >= 2
    _sched(A, ctx, snap, flags=1 | A.ANDES_DEBUG_CHECKS)
    _expect_next_call_fails(A, ctx, A.ANDES_E_RANGE)


def test_debug_checks_off_do_not_report(A, ctx):
    _sched(A, ctx, _bad("rank"), flags=1)
    _sched(A, ctx, W.random_small(1, n=5))


def test_host_entry_rejects_null_arrays(A, ctx):
    snap = W.random_small(4, n=10)
    hreq = A.requests_to(snap, pin=True)
    tau_h = torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).pin_memory()
    for k in ("ttft_us", "rank", "running", "tl_pool"):
        bad = dict(hreq, **{k: None})
        with pytest.raises(A.AndesError) as ei:
            ctx.schedule_host(bad, snap.n, snap.now_us, snap.horizon_us, tau_h, snap.kv_capacity)
        assert ei.value.rc == A.ANDES_E_INVAL
    out, rc = ctx.schedule_host(hreq, snap.n, snap.now_us, snap.horizon_us, tau_h, snap.kv_capacity)
    assert rc in (0, 1)
