import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


# Full-size snapshots and their oracle decisions, shared by the headline parity tests
# (tests/test_gpu_headline.py, tests/test_gpu_shard.py): the oracle's per-B walks run on every
# host core (oracle.schedule(threads=...), outputs independent of the split).
_SNAPS = {}
_ORC_DEC = {}


def snapshot_cached(name):
    import workloads as W
    if name not in _SNAPS:
        _SNAPS[name] = {"config2": W.config2, "config3": W.config3, "config4": W.config4}[name]()
    return _SNAPS[name]


def oracle_decision_cached(orc, name, snap, cap=None, flags=1, cur_latency=0, prefill=5000, swap=0):
    cap = snap.preempt_cap if cap is None else cap
    key = (name, cap, flags, cur_latency, prefill, swap)
    if key not in _ORC_DEC:
        _ORC_DEC[key] = orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity,
                                     preempt_cap=cap, cur_latency_us=cur_latency, flags=flags,
                                     prefill_tok_s=prefill, swap_tok_s=swap, threads=orc.nproc())
    return _ORC_DEC[key]


def assert_decision_equal(g, o):
    """A GPU decision (dict of numpy arrays: mask, admit, preempt, sc, V, kstar) against an
    oracle decision: every output, the admit list in greedy order and the preempt list in
    victim order (BASELINE north_star: bit-exact selections)."""
    import numpy as np
    assert bool(g["sc"][6] & 1) == (o.status == 0)
    np.testing.assert_array_equal(g["mask"], o.serve_mask)
    if o.status != 0:
        return
    assert [int(x) for x in g["sc"][[0, 1, 2, 3, 4, 5, 7]]] == [o.B_star, o.realized, o.admit.size, o.preempt.size,
                                                                o.B_lo, o.B_hi, o.k_star]
    assert int(g["sc"][6]) & 39 == o.flags & 39
    np.testing.assert_array_equal(g["V"], o.V)
    np.testing.assert_array_equal(g["kstar"], o.kstar)
    np.testing.assert_array_equal(g["admit"], o.admit)
    np.testing.assert_array_equal(g["preempt"], o.preempt)
