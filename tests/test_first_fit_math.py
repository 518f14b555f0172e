"""The identity behind k_mc_lane's exact first fit (DESIGN "k_mc_lane"), checked on random
feasible profiles against brute force -- the math, independent of any kernel.

For a head (s, w) with L = M - s and a projected profile Prof(t+u), u >= 1 (zero past its
end), the head fits at offset D iff Prof(t+D+tau) + s + tau <= M for tau = 1..w (Eq. 5 with
the profile only advancing).  With c_u = max(0, min(u, Prof(t+u) + u - L)) and
F(x) = max_{u <= x} c_u:  feasible(D) <=> F(D + w) <= D, and the first feasible D is the
least fixpoint of D <- F(D + w) from D = 0.
"""
import numpy as np


def brute_first_fit(prof, s, w, M):
    D = 0
    while True:
        if all((prof[D + tau] if D + tau < len(prof) else 0) + s + tau <= M for tau in range(1, w + 1)):
            return D
        D += 1


def fixpoint_first_fit(prof, s, w, M, width):
    L = M - s
    c = [0] + [max(0, min(u, (prof[u] if u < len(prof) else 0) + u - L)) for u in range(1, width + 1)]
    F = np.maximum.accumulate(c)
    D = 0
    while True:
        f = F[min(D + w, width)]
        if f <= D:
            return D
        D = int(f)


def random_profile(g, M, horizon):
    """Sum of ramps s_j + k (k = 1..o_j) of requests started at or before t (Eq. 3), kept
    feasible (<= M) like MC-SF's admissions keep it."""
    prof = np.zeros(horizon + 1, dtype=np.int64)
    for _ in range(g.integers(0, 12)):
        s = int(g.integers(1, max(2, M // 6)))
        o = int(g.integers(1, M - s + 1))
        started = int(g.integers(0, o))            # rounds already run
        ramp = np.zeros_like(prof)
        for u in range(1, o - started + 1):
            ramp[u] = s + started + u
        if (prof + ramp <= M).all():
            prof += ramp
    return prof


def test_fixpoint_equals_brute_force_first_fit():
    g = np.random.default_rng(2502)
    for _ in range(3000):
        M = int(g.integers(4, 65))
        prof = random_profile(g, M, 64)
        s = int(g.integers(1, M))
        w = int(g.integers(1, M - s + 1))
        assert fixpoint_first_fit(prof, s, w, M, 64) == brute_first_fit(prof, s, w, M)


def test_feasibility_characterisation():
    g = np.random.default_rng(7115)
    for _ in range(1000):
        M = int(g.integers(4, 65))
        prof = random_profile(g, M, 64)
        s = int(g.integers(1, M))
        w = int(g.integers(1, M - s + 1))
        L = M - s
        c = [0] + [max(0, min(u, (prof[u] if u < len(prof) else 0) + u - L)) for u in range(1, 200)]
        F = np.maximum.accumulate(c)
        for D in range(0, 70):
            direct = all((prof[D + tau] if D + tau < len(prof) else 0) + s + tau <= M for tau in range(1, w + 1))
            assert direct == (F[D + w] <= D), (M, s, w, D)
