"""CPU check of the case analysis behind the scan's pass-2 skip (scan.cu, warp_tile_aligned,
two-tile units): a plain-Python model of one lane's arithmetic -- pass 1's
unclamped zero-carry sum, then the closed form (carry >= dz, or a constant zero-carry lateness),
s0 (carry <= L1), the walk up to the first token whose zero-carry consumption reaches I + carry,
or the lane's own clamped walk -- against the literal recurrence A_j = max(A_{j-1} + P, d_j),
sum of min(A_j, t) - I_j (Eq. 1 over a sub-range with a carried lateness; reading R2).  This pins
the derivation, not the kernel: the kernel itself is compared with the oracle by the -m gpu
tests (test_scan_unit_width_forced)."""
import random


def literal(d, Is, P, c, t):
    A, s = Is - P + c, 0
    for j, x in enumerate(d):
        A = max(A + P, x)
        s += min(A, t) - (Is + j * P)
    return s, A


def lane_model(d, Is, P, c, t, final=False):
    n, a, s0 = len(d), Is - P, 0
    for x in d:  # pass 1: zero-carry recurrence, unclamped sum
        a = max(a + P, x)
        s0 += a
    dz = a - (Is + (n - 1) * P)
    L1 = max(d[0], Is) - Is
    Ilast = Is + (n - 1) * P
    sumI = n * Is + P * n * (n - 1) // 2
    edge = Ilast + max(c, dz)  # the last token's consumption time
    if c >= dz or L1 >= dz:  # A_j = I_j + max(c, dz) at every token: closed form
        Lc = max(c, dz)
        b0 = Is + Lc
        if b0 + (n - 1) * P <= t:
            k = n
        elif b0 > t:
            k = 0
        else:
            k = min(n, (t - b0) // P + 1)
        return k * Lc + (n - k) * (t - Is) - P * (n * (n - 1) // 2 - k * (k - 1) // 2), edge
    if not final and Ilast + max(c, dz) > t:  # some token clamps: the lane walks with the carry
        Ac, sc = Is - P + c, 0
        for x in d:
            Ac = max(Ac + P, x)
            sc += min(Ac, t)
        return sc - sumI, edge
    fix = 0
    if c > L1:  # walk up to the first token whose zero-carry consumption reaches I + c
        A0, Ic = Is - P, Is - P + c
        for x in d:
            A0, Ic = max(A0 + P, x), Ic + P
            if A0 >= Ic:
                break
            fix += Ic - A0
    return s0 + fix - sumI, edge


def test_lane_model_equals_literal_recurrence():
    rng = random.Random(7)
    for _ in range(40000):
        n = rng.randint(1, 14)
        P = rng.randint(1, 60)
        Is = rng.randint(0, 400)
        x, d = rng.randint(0, 500), []
        kind = rng.randrange(3)
        for j in range(n):
            # nondecreasing deliveries: behind schedule, ahead of it (constant lateness), mixed
            x += rng.randint(0, 2 * P) if kind == 0 else rng.randint(0, P // 2) if kind == 1 else rng.randint(0, 90)
            d.append(x)
        c = rng.choice([0, rng.randint(0, 400)])
        t = Is + (n - 1) * P + rng.choice([0, rng.randint(0, 600)])  # every token due: I_j <= t
        want, A_last = literal(d, Is, P, c, t)
        got, edge = lane_model(d, Is, P, c, t)
        assert got == want, (d, Is, P, c, t)
        assert edge == A_last  # the edge value: the last token's consumption time
        want_f, _ = literal(d, Is, P, c, 1 << 62)
        assert lane_model(d, Is, P, c, 1 << 62, final=True)[0] == want_f
