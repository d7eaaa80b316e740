"""andes_simulate (-m gpu; NEXT-3): the serving loop on the device with the decision in the loop,
against the same loop on the host with the CPU oracle's decision (tests/sim_reference.py): every
request's delivered-token count and every delivery time identical, the same iteration count;
for Andes' priority and for LQSF (reading R21), with and without contention."""
import numpy as np
import pytest

import workloads as W
from sim_reference import simulate_reference

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    import paper_2404_16283_b200 as A
    from paper_2404_16283_b200 import build
    build.build()
    return A


@pytest.mark.parametrize("seed,rho,flags,M,cap", [(1, 1.0, 0, 20_000, W.UINT32_MAX), (2, 1.5, 16, 12_000, W.UINT32_MAX),
                                                  (3, 0.6, 0, 60_000, 2), (4, 2.0, 16, 15_000, 1)])
def test_simulate_equals_host_loop_with_oracle(A, orc, seed, rho, flags, M, cap):
    tr = W.sim_trace(seed, rho, window_s=12.0, rate_at_rho1=2.5, max_prompt=3000, max_out=40)
    tau = W.tau_table(16)
    ctx = A.Context(max_requests=tr["n"], max_B=16, max_tokens=tr["tl_len"] + 64)
    taud = torch.from_numpy(tau.view(np.int32)).cuda()
    g, pool, t, st = ctx.simulate(tr, taud, M, preempt_cap=cap, flags=flags)
    torch.cuda.synchronize()
    rg, rtl, rit = simulate_reference(orc, tr, tau, M, preempt_cap=cap, flags=flags)
    assert st["iterations"] == rit and st["finished"] == tr["n"]
    gg = g.cpu().numpy()
    np.testing.assert_array_equal(gg, rg)
    pool = pool.cpu().numpy().view(np.uint32)
    for i in range(tr["n"]):
        b = int(tr["tl_base"][i])
        np.testing.assert_array_equal(pool[b:b + gg[i]], np.asarray(rtl[i], np.uint32))
    assert (gg == tr["output_len"]).all()
