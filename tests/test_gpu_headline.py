"""Oracle parity at the headline sizes (-m gpu; slow): the full BASELINE config-3 decision
(65,536 requests, B = 1..256, preemption cap 16) and the config-4 population (2^20 requests)
through the C ABI, compared element by element with the CPU oracle's literal decision
(oracle.schedule, Algorithm 1 per B with a full sort and `break`; its per-B walks
run on every host core, which leaves every output unchanged).

Compared: every scalar (B*, realized, n_admit, n_preempt, B_lo, B_hi, flags, k*(B*)), V(B) and
k*(B) for all 256 B, the whole serve mask, and the admit and preempt lists IN ORDER; gains and
keys of every request at a spread of B (bit-equal fp64 / fp32)."""
import numpy as np
import pytest

import workloads as W
from conftest import assert_decision_equal, oracle_decision_cached, snapshot_cached

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


@pytest.fixture(scope="module")
def ctx3(A):
    return A.Context(max_requests=1 << 16, max_B=256, max_tokens=1 << 24, max_running=4096)


def _tau(snap):
    return torch.from_numpy(np.asarray(snap.tau_us, np.uint32).view(np.int32)).cuda()


def _gpu_decision(A, ctx, snap, cap, flags, prefill=5000, swap=0):
    d = ctx.schedule(A.requests_to(snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), snap.kv_capacity,
                     preempt_cap=cap, flags=flags, prefill_tok_s=prefill, swap_tok_s=swap)
    torch.cuda.synchronize()
    sc = d.scalars.cpu().numpy().view(np.uint32).copy()
    return dict(mask=d.serve_mask.cpu().numpy()[:snap.n], admit=d.admit.cpu().numpy().view(np.uint32)[:sc[2]],
                preempt=d.preempt.cpu().numpy().view(np.uint32)[:sc[3]], sc=sc, V=d.V.cpu().numpy(),
                kstar=d.kstar.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("flags,cap", [(1, 16), (1, W.UINT32_MAX), (1 | 16, 16), (1 | 32, 16), (1 | 64, 16),
                                       (1 | 128, 16), (1 | 2, 16)],
                         ids=["andes-cap16", "andes-nocap", "lqsf", "maxmin", "perfect", "refine", "pruned"])
def test_config3_decision_equals_oracle(A, ctx3, orc, flags, cap):
    """BASELINE config 3 (the bench workload, same entry point) against the oracle: the Andes
    decision with and without the cap, the LQSF priority (R21), both Appendix-A objectives
    (R22-R23), the overhead-aware refiner (R24-R27) and B-range pruning."""
    snap = snapshot_cached("config3")
    o = oracle_decision_cached(orc, "config3", snap, cap=cap, flags=flags)
    g = _gpu_decision(A, ctx3, snap, cap, flags)
    assert_decision_equal(g, o)
    if flags == 1 and cap == 16:
        assert o.B_hi == 256 and o.flags & 2  # the cap binds on the headline workload
        g2 = _gpu_decision(A, ctx3, snap, cap, flags)  # deterministic
        for k in g:
            np.testing.assert_array_equal(g[k], g2[k])


def test_config3_gains_every_request(A, ctx3, orc):
    """S3 on all 65,536 requests at 16 B values spread over 1..256 (incl. the B_lo crossings of
    both reading speeds, 235/236): fp64 gains, Q_wait and fp32 keys bit-equal."""
    snap = snapshot_cached("config3")
    Bl = np.array([1, 2, 3, 16, 38, 64, 100, 127, 128, 170, 200, 234, 235, 236, 255, 256])
    gain, key, qw = ctx3.gain_estimate(A.requests_to(snap), snap.n, snap.now_us, snap.horizon_us, _tau(snap), Bl)
    torch.cuda.synchronize()
    og, ok, oqw = orc.gain_estimate(snap, snap.now_us, snap.horizon_us, snap.tau_us, Bl, threads=orc.nproc())
    np.testing.assert_array_equal(qw.cpu().numpy(), oqw)
    np.testing.assert_array_equal(gain.cpu().numpy(), og)
    np.testing.assert_array_equal(key.cpu().numpy().view(np.uint32), ok.view(np.uint32))


def test_config4_decision_equals_oracle(A, orc):
    """BASELINE config 4's population (2^20 live requests, 140 M timestamps) on one GPU through
    andes_schedule and through the sharded entry point at world 1, against the oracle."""
    from test_gpu_shard import run_sharded
    snap = snapshot_cached("config4")
    o = oracle_decision_cached(orc, "config4", snap, cap=16, flags=1)
    ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64, max_running=4096)
    g = _gpu_decision(A, ctx, snap, 16, 1)
    assert_decision_equal(g, o)
    del ctx
    r = run_sharded(A, snap, 1, cap=16)[0]
    assert_decision_equal(r, o)


@pytest.mark.parametrize("G", [2, 8])
def test_config4_sharded_equals_oracle(A, orc, G):
    """Config 4 split into G contiguous shards (the multi-GPU decision's five steps run in
    lockstep on one GPU, the four all-gathers as device copies in rank order) against the oracle:
    every rank holds the same replicated outputs; the serve masks concatenate to the oracle's."""
    from test_gpu_shard import run_sharded
    snap = snapshot_cached("config4")
    o = oracle_decision_cached(orc, "config4", snap, cap=16, flags=1)
    res = run_sharded(A, snap, G, cap=16)
    mask = np.concatenate([r["mask"] for r in res])
    for r in res:
        assert_decision_equal(dict(r, mask=mask), o)
