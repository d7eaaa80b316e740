"""Config 1 (-m "not gpu"): the 200-iteration driver on the oracle with brute force bounding
Algorithm 1 at every candidate B of every iteration (SPEC acceptance: greedy <=
exact), and the greedy/exact ratio of the chosen decision."""
from config1 import QualityTracker, run


def test_config1_greedy_bounded_by_exact_every_iteration(orc):
    qt = QualityTracker(orc)

    def decide(snap):
        return orc.schedule(snap, snap.now_us, snap.horizon_us, snap.tau_us, snap.kv_capacity)

    assert run(decide, on_iter=qt) >= 150
    s = qt.summary()
    assert s["B_values_checked"] >= 150
    assert 0.0 < s["ratio_min"] <= 1.0 and s["ratio_mean"] <= 1.0
    print(s)
