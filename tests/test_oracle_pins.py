"""Pins for the CPU oracle (oracle/), checked against what the paper and mathematics fix.

Each pin is independent of the oracle's own code: values printed or worked from the paper
(tests/golden/), closed forms, invariants of the model (Eq. 3), special
cases that reduce to something known, published RNG known-answer vectors, a brute-force
optimum cross-checked against an independent MILP solve of Eqs. 1-4 (scipy/HiGHS).
"""
import json
from pathlib import Path

import numpy as np
import pytest

import workloads as W

GOLDEN = Path(__file__).resolve().parent / "golden"
POL = {"mcsf": 0, "mcbench": 1, "alpha": 2, "alpha_beta": 3}


# ----------------------------------------------------------------------------------------
# independent checkers written from the model, not from the oracle
# ----------------------------------------------------------------------------------------
def memory_profile(req, start):
    """Eq. 3: a request started at k holds s + t - k at t = k+1..k+o."""
    req = np.asarray(req)
    horizon = int(max((start[i] + req[i, 2] for i in range(len(req))), default=0)) + 2
    prof = np.zeros(horizon + 1, dtype=np.int64)
    for i in range(len(req)):
        k, s, o = int(start[i]), int(req[i, 1]), int(req[i, 2])
        for t in range(k + 1, k + o + 1):
            prof[t] += s + t - k
    return prof


def check_schedule(req, M, out):
    """Validity of a completed schedule under the model."""
    req = np.asarray(req)
    p, c = out["start"], out["completion"]
    assert (p >= req[:, 0]).all(), "start before arrival (Eq. 2 sums from a_i)"
    assert (c == p + req[:, 2]).all(), "non-preemptive: c = p + o (P:88)"
    prof = memory_profile(req, p)
    assert prof.max(initial=0) <= M, "memory constraint Eq. 3 violated"
    # TEL and Little's law: TEL = sum_t N(t), N(t) = #{i: a_i <= t < c_i}
    tel = int((c - req[:, 0]).sum())
    assert out["tel"] == tel
    N = np.zeros(int(c.max(initial=0)) + 2, dtype=np.int64)
    for i in range(len(req)):
        N[req[i, 0]:c[i]] += 1
    assert N.sum() == tel
    assert out["rounds"] == int((N > 0).sum())
    assert out["makespan"] == int(c.max(initial=0))
    return prof


# ----------------------------------------------------------------------------------------
def test_philox_known_answers(oracle_mod):
    """Random123 kat_vectors for philox4x32_10 (Salmon et al., SC'11)."""
    O = oracle_mod
    assert O.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_eq5_direct_evaluation_examples(oracle_mod):
    """Eq. 5 evaluated by hand."""
    O = oracle_mod
    # S empty, U = two (s=1, o~=2) at t=0, t'=2: 3 + 3
    assert O.projected_occupancy(2, 0, [], [(1, 2), (1, 2)]) == 6
    # S = {(s=2, p=0, o~=3)}, t=1: t'=3 -> 2+3; t'=4 -> indicator off
    assert O.projected_occupancy(3, 1, [(2, 0, 3)], []) == 5
    assert O.projected_occupancy(4, 1, [(2, 0, 3)], []) == 0
    assert O.is_feasible(0, 6, [], [(1, 2), (1, 2)]) is True
    assert O.is_feasible(0, 5, [], [(1, 2), (1, 2)]) is False
    # U empty: range [t+1, t_max(U)] is empty -> feasible
    assert O.is_feasible(3, 0, [(5, 0, 9)], []) is True


def test_checkpoint_sufficiency_fuzz(oracle_mod):
    """checking Eq. 5 only at the completion times p_j + o~_j of S u U is enough,
    because memory grows linearly between completions.  The oracle scans every t';
    here an independent checkpoint-only evaluation must agree on random queries."""
    O = oracle_mod
    g = np.random.default_rng(11)
    for _ in range(400):
        t = int(g.integers(0, 30))
        S = [(int(g.integers(1, 6)), int(t - g.integers(0, 8)), int(g.integers(1, 15))) for _ in range(g.integers(0, 5))]
        S = [(s, p, op) for (s, p, op) in S if p + op > t]          # still projected-active
        U = [(int(g.integers(1, 6)), int(g.integers(1, 15))) for _ in range(g.integers(1, 5))]
        budget = int(g.integers(5, 60))
        tmax = max(t + op for _, op in U)
        cps = sorted({p + op for (_, p, op) in S} | {t + op for (_, op) in U})
        cps = [c for c in cps if t + 1 <= c <= tmax]

        def load(tp):
            return sum(s + tp - p for (s, p, op) in S if op >= tp - p) + \
                sum(s + tp - t for (s, op) in U if op >= tp - t)
        cp_ok = all(load(c) <= budget for c in cps)
        assert O.is_feasible(t, budget, S, U) == cp_ok


@pytest.mark.parametrize("case", json.loads((GOLDEN / "worked_examples.json").read_text())["cases"],
                         ids=lambda c: c["name"])
def test_worked_examples(oracle_mod, case):
    O = oracle_mod
    alpha = tuple(case.get("alpha", (0, 1)))
    out = O.simulate(case["req"], case["M"], POL[case["policy"]], alpha=alpha)
    for k, v in case["expect"].items():
        got = out[k]
        if isinstance(v, list):
            assert list(got) == v, (k, list(got), v)
        else:
            assert got == v, (k, got, v)
    if "opt" in case:
        opt, _, _ = O.opt_bruteforce(case["req"], case["M"])
        assert opt == case["opt"]


@pytest.mark.parametrize("s,o,m,k", [(2, 3, 2, 3), (1, 1, 3, 4), (3, 5, 4, 2), (1, 7, 1, 5), (2, 2, 5, 3)])
def test_identical_requests_closed_form(oracle_mod, s, o, m, k):
    """n = k*m identical (s, o) at 0 with M = m(s+o): k back-to-back batches of m
    (cf. the batch arithmetic of P:744-748): TEL = o m k(k+1)/2, makespan k o."""
    O = oracle_mod
    out = O.simulate([[0, s, o, o]] * (k * m), m * (s + o))
    assert out["tel"] == o * m * k * (k + 1) // 2
    assert out["makespan"] == k * o


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_unconstrained_memory(oracle_mod, policy):
    """If M >= sum_i (s_i + o_i) nothing ever waits: c_i = a_i + o_i, TEL = sum o."""
    O = oracle_mod
    b = W.random_small(40, seed=3, n_max=12, M_lo=4, M_hi=30)
    for k in range(b.n_inst):
        req, _ = b.instance(k)
        if len(req) == 0:
            continue
        M = int((req[:, 1] + req[:, 2]).sum())
        out = O.simulate(req, M, policy, alpha=(1, 1000000), beta_thresh=2**31, seed=1)
        assert out["status"] == 0
        assert (out["completion"] == req[:, 0] + req[:, 2]).all()
        assert out["tel"] == int(req[:, 2].sum())
        assert out["evictions"] == 0


def test_volume_identity(oracle_mod):
    """A request of (s, o) running alone occupies vol_o = s o + o(o+1)/2 slot-rounds
    (P:212); peak s + o."""
    O = oracle_mod
    for s in range(1, 6):
        for o in range(1, 12):
            out = O.simulate([[3, s, o, o]], s + o)
            prof = memory_profile([[3, s, o, o]], out["start"])
            assert prof.sum() == s * o + o * (o + 1) // 2
            assert out["peak"] == s + o == prof.max()


@pytest.mark.parametrize("maker", ["c1a", "c1b", "fuzz", "am2"])
@pytest.mark.parametrize("policy", [0, 1])
def test_mc_schedules_valid(oracle_mod, maker, policy):
    """Every MC-SF / MC-Benchmark schedule satisfies the model: p >= a, c = p + o,
    memory <= M every round (Eq. 3), TEL = sum_t N(t), peak = max memory."""
    O = oracle_mod
    b = {"c1a": lambda: W.c1(150, 7, "a"), "c1b": lambda: W.c1(150, 7, "b"),
         "fuzz": lambda: W.random_small(150, 5), "am2": lambda: W.am2(60, 9)}[maker]()
    for k in range(b.n_inst):
        req, M = b.instance(k)
        out = O.simulate(req, M, policy)
        assert out["status"] == 0
        if len(req) == 0:
            assert out["tel"] == 0 and out["rounds"] == 0
            continue
        prof = check_schedule(req, M, out)
        assert out["peak"] == prof.max()


def _rank_key(req, policy, i):
    return (int(req[i, 3]), i) if policy == 0 else (i,)


@pytest.mark.parametrize("policy", [0, 1])
def test_prefix_maximality(oracle_mod, policy):
    """Alg. 1/2: at every round the started set is a prefix of the waiting queue in key
    order, feasible, and the next waiting request would violate Eq. 5."""
    O = oracle_mod
    b = W.random_small(80, 21, n_max=16, M_lo=6, M_hi=40, a_max=12)
    for k in range(b.n_inst):
        req, M = b.instance(k)
        n = len(req)
        if n == 0:
            continue
        out = O.simulate(req, M, policy)
        p, c = out["start"], out["completion"]
        proj = req[:, 3] if policy == 0 else req[:, 2]
        for t in sorted(set(range(int(req[0, 0]), int(c.max()) + 1))):
            R = [i for i in range(n) if req[i, 0] <= t <= p[i]]
            if not R:
                continue
            R.sort(key=lambda i: _rank_key(req, policy, i))
            U = [i for i in R if p[i] == t]
            assert R[:len(U)] == U, "admitted set is not a prefix"
            if len(U) < len(R):
                S = [(int(req[j, 1]), int(p[j]), int(proj[j])) for j in range(n) if p[j] < t < c[j]]
                Ul = [(int(req[i, 1]), int(proj[i])) for i in R[:len(U) + 1]]
                assert not O.is_feasible(t, M, S, Ul), "next candidate was feasible"


def test_mcbench_equals_mcsf_when_orders_coincide(oracle_mod):
    """Alg. 2 differs from Alg. 1 only in the order of R; if arrival order equals the
    o~ order the schedules coincide."""
    O = oracle_mod
    b = W.random_small(100, 31, n_max=20, M_lo=8, M_hi=50, a_max=0)
    for k in range(b.n_inst):
        req, M = b.instance(k)
        req = req[np.argsort(req[:, 3], kind="stable")]
        x, y = O.simulate(req, M, 0), O.simulate(req, M, 1)
        assert (x["completion"] == y["completion"]).all()


def test_beta_one_is_alpha_greedy(oracle_mod):
    """beta = 1 (threshold 2^32) clears every active request: the alpha-greedy rule."""
    O = oracle_mod
    b = W.c4(6, 41)
    for k in range(b.n_inst):
        req, M = b.instance(k)
        x = O.simulate(req, M, 2, alpha=(1, 10))
        y = O.simulate(req, M, 3, alpha=(1, 10), beta_thresh=2**32, seed=99)
        for key in ("completion", "tel", "evictions", "status", "peak"):
            assert np.array_equal(np.asarray(x[key]), np.asarray(y[key]))


def test_alpha_beta_deterministic_and_seeded(oracle_mod):
    O = oracle_mod
    b = W.random_small(40, 43, n_max=30, M_lo=20, M_hi=60, a_max=10)
    k = max(range(b.n_inst), key=lambda k: O.simulate(*b.instance(k), 3, alpha=(1, 10),
                                                      beta_thresh=W.beta_threshold(0.2), seed=5)["evictions"])
    req, M = b.instance(k)
    x = O.simulate(req, M, 3, alpha=(1, 10), beta_thresh=W.beta_threshold(0.2), seed=5)
    y = O.simulate(req, M, 3, alpha=(1, 10), beta_thresh=W.beta_threshold(0.2), seed=5)
    z = O.simulate(req, M, 3, alpha=(1, 10), beta_thresh=W.beta_threshold(0.2), seed=6)
    assert np.array_equal(x["completion"], y["completion"])
    assert x["evictions"] > 0
    assert not np.array_equal(x["completion"], z["completion"])


def test_alpha_livelock_and_stuck(oracle_mod):
    O = oracle_mod
    # E9 cycle with a short cap: evicted at 24, re-admitted at 25, cap 30 -> LIVELOCK
    out = O.simulate([[0, 1, 40, 40], [0, 1, 40, 40]], 50, 2, alpha=(3, 10), round_cap=30)
    assert out["status"] == 2 and out["evictions"] == 2 and list(out["start"]) == [25, 25]
    # head-of-line request needs s+1 = 21 > B = floor(0.4*50) = 20 on an empty worker
    out = O.simulate([[0, 20, 5, 5], [0, 1, 4, 4]], 50, 2, alpha=(6, 10))
    assert out["status"] == 2 and out["decision_rounds"] == 1
    # beta-clearing breaks the E9 cycle
    out = O.simulate([[0, 1, 40, 40], [0, 1, 40, 40]], 50, 3, alpha=(3, 10), beta_thresh=2**31, seed=7)
    assert out["status"] == 0 and out["evictions"] > 0


def test_invalid_instances(oracle_mod):
    O = oracle_mod
    assert O.simulate([[0, 5, 6, 6]], 10, 0)["status"] == 1            # s + o~ > M
    assert O.simulate([[0, 5, 6, 6]], 10, 2, alpha=(1, 4))["status"] == 1
    assert O.simulate([[3, 1, 1, 1], [2, 1, 1, 1]], 10, 0)["status"] == 1   # unsorted a
    assert O.simulate([[0, 0, 1, 1]], 10, 0)["status"] == 1            # s < 1
    assert O.simulate([[0, 1, 3, 2]], 10, 0)["status"] == 1            # o~ < o
    out = O.simulate(np.zeros((0, 4), np.int32), 10, 0)
    assert out["status"] == 0 and out["tel"] == 0 and out["rounds"] == 0


def test_prediction_overestimate_mcsf(oracle_mod):
    """MC-SF with o~ >= o: memory-safe (Eq. 3 <= M) and completes at p + o."""
    O = oracle_mod
    b = W.random_small(120, 51, n_max=20, M_lo=10, M_hi=60, pred_slack=6)
    assert (b.req[:, 3] >= b.req[:, 2]).all() and (b.req[:, 3] > b.req[:, 2]).any()
    for k in range(b.n_inst):
        req, M = b.instance(k)
        out = O.simulate(req, M, 0)
        assert out["status"] == 0
        if len(req):
            check_schedule(req, M, out)


# ----------------------------------------------------------------------------------------
# hindsight optimum: brute force vs an independent MILP of Eqs. 1-4
# ----------------------------------------------------------------------------------------
def milp_opt(req, M, horizon):
    """Eqs. 1-4 solved with scipy.optimize.milp (HiGHS)."""
    from scipy.optimize import LinearConstraint, milp
    from scipy.sparse import lil_matrix
    req = np.asarray(req)
    n = len(req)
    var = []
    for i in range(n):
        for t in range(int(req[i, 0]), horizon + 1):
            var.append((i, t))
    nv = len(var)
    cost = np.array([t for (_, t) in var], dtype=float)
    const = float((req[:, 2] - req[:, 0]).sum())
    T_mem = horizon + int(req[:, 2].max()) + 1
    A = lil_matrix((n + T_mem, nv))
    lb = np.zeros(n + T_mem)
    ub = np.zeros(n + T_mem)
    for v, (i, t) in enumerate(var):
        A[i, v] = 1.0                                     # Eq. 2
        s, o = int(req[i, 1]), int(req[i, 2])
        for tt in range(t + 1, t + o + 1):               # Eq. 3: active at t+1..t+o
            A[n + tt - 1, v] = s + tt - t
    lb[:n] = 1
    ub[:n] = 1
    lb[n:] = -np.inf
    ub[n:] = M
    res = milp(cost, constraints=LinearConstraint(A.tocsr(), lb, ub),
               integrality=np.ones(nv), bounds=(0, 1))
    assert res.status == 0
    return int(round(res.fun + const))


def test_bruteforce_opt_matches_milp(oracle_mod):
    O = oracle_mod
    pytest.importorskip("scipy")
    cases = [W.c1(12, 61, "a"), W.c1(12, 61, "b")]
    for b in cases:
        for k in range(b.n_inst):
            req, M = b.instance(k)
            ub = O.simulate(req, M, 0)["tel"]
            opt, _, _ = O.opt_bruteforce(req, M, ub)
            horizon = int(req[:, 0].max()) + ub
            assert opt == milp_opt(req, M, horizon)
    # the Thm 1 instance variant where MC-SF is not optimal (E7, r = 13)
    req = [[0, 1, 15, 15]] + [[13, 1, 1, 1]] * 8
    assert milp_opt(req, 16, 13 + 39) == 35


def test_mcsf_never_beats_opt_and_lb(oracle_mod):
    """North-star invariant: TEL(MC-SF) >= OPT on every tiny instance; LB_sorted <= OPT
    on all-at-0 instances; the returned optimal start vector is itself a valid schedule."""
    O = oracle_mod
    for variant in ("a", "b"):
        b = W.c1(300, 71, variant)
        for k in range(b.n_inst):
            req, M = b.instance(k)
            mc = O.simulate(req, M, 0)["tel"]
            opt, st, _ = O.opt_bruteforce(req, M, mc)
            assert opt <= mc
            if variant == "a":
                assert O.lb_sorted(req, M) <= opt
            if st is not None:
                prof = memory_profile(req, st)
                assert prof.max() <= M and (st >= req[:, 0]).all()
                assert int((st + req[:, 2] - req[:, 0]).sum()) == opt


def test_lb_sorted_closed_form(oracle_mod):
    """LB_sorted of identical requests (s, o) at 0: V_k = k vol, c_(k) >= max(ceil(k vol/M), o)."""
    O = oracle_mod
    s, o, n, M = 2, 3, 6, 10
    vol = s * o + o * (o + 1) // 2
    expect = sum(max(-(-k * vol // M), o) for k in range(1, n + 1))
    assert O.lb_sorted([[0, s, o, o]] * n, M) == expect


def test_policy_ordering_table1_shape(oracle_mod):
    """Table 1 orders MC-SF < MC-Benchmark < every alpha / alpha-beta row.
    In unit rounds on the trace-shaped C4 workload the same ordering must hold."""
    O = oracle_mod
    b = W.c4(12, 81)
    means = {}
    for name, pol, alpha, beta in W.C4_POLICIES:
        out = O.simulate_batch(b.offset, b.req, b.mem, POL[pol], alpha=alpha or (0, 1),
                               beta_thresh=W.beta_threshold(beta or 0.0), seed=1)
        ok = out["status"] == 0
        means[name] = float(out["tel"][ok].sum() / (1000 * ok.sum()))
    assert means["MC-SF"] < means["MC-Benchmark"]
    for name in means:
        if name.startswith("alpha"):
            assert means["MC-Benchmark"] < means[name]


# ----------------------------------------------------------------------------------------
# NEXT-1: MC-SF under prediction error with a protection margin
# ----------------------------------------------------------------------------------------
def test_protected_mcsf_reduces_to_mcsf(oracle_mod):
    """alpha = 0 and o^ >= o: the projection never underestimates, nothing overflows, so
    the protected variant is Algorithm 1 with o~ = o^."""
    O = oracle_mod
    small = W.random_small(120, 91, n_max=25, M_lo=8, M_hi=60, a_max=20, pred_slack=5)
    # budgets past 64 as well: the CUDA ring path runs MC-SF with o~ > o this way
    large = W.random_small(60, 93, n_max=40, M_lo=65, M_hi=400, a_max=30, pred_slack=40)
    insts = [small.instance(k) for k in range(small.n_inst)] + [large.instance(k) for k in range(large.n_inst)]
    b = W.from_instances(insts)
    assert (b.req[:, 3] > b.req[:, 2]).any() and (b.mem > 64).any()
    for k in range(b.n_inst):
        req, M = b.instance(k)
        x, y = O.simulate(req, M, O.MCSF), O.simulate(req, M, O.MCSF_PROT, alpha=(0, 1))
        for key in ("completion", "tel", "status", "peak", "decision_rounds"):
            assert np.array_equal(np.asarray(x[key]), np.asarray(y[key]))
        assert y["evictions"] == 0


def test_protected_mcsf_overflow_worked_example(oracle_mod):
    """Two (s=1, o=6) requests predicted o^=2, M=10, alpha=0: both start at 0 (projection
    peaks at 6); the realised memory reaches 10 at t=4 and 12 at t=5, so round 4 clears
    both; re-admitted at 5, cleared again at 9 with nothing completed or arrived:
    the cycle repeats for ever (DESIGN Q24).  With a third request arriving at 7 the second
    clear is not a repeat; the third clear at 11 is."""
    O = oracle_mod
    r = O.simulate([[0, 1, 6, 2], [0, 1, 6, 2]], 10, O.MCSF_PROT, alpha=(0, 1))
    assert (r["status"], r["decision_rounds"], r["evictions"], r["peak"]) == (2, 2, 4, 10)
    r = O.simulate([[0, 1, 6, 2], [0, 1, 6, 2], [7, 1, 3, 3]], 10, O.MCSF_PROT, alpha=(0, 1))
    assert (r["status"], r["decision_rounds"], r["evictions"], r["peak"]) == (2, 4, 8, 10)
    # alpha = 0.5 (budget 5): A starts at 0; B fails at t=1? no -- A's projection ends at
    # t'=2 (o^=2), so at t=1 B's window sees 3+2=5 at t'=2 and 3 at t'=3: B starts at 1.
    # Realised Mem(5) = 6 + 5 = 11 > 10 at t=4: clear; A at 5, B at 6, clear at 9 (repeat).
    # Decision rounds t = 0, 1, 5, 6; peak Mem(4) = 5 + 4 = 9.
    r = O.simulate([[0, 1, 6, 2], [0, 1, 6, 2]], 10, O.MCSF_PROT, alpha=(1, 2))
    assert (r["status"], r["decision_rounds"], r["evictions"], r["peak"]) == (2, 4, 4, 9)


@pytest.mark.parametrize("eps", [0.2, 0.5, 0.8])
def test_protected_mcsf_schedules_valid(oracle_mod, eps):
    """Every completed protected-MC-SF schedule respects the model (p >= a, c = p + o,
    memory <= M every round): clearing removes any batch that would overflow."""
    O = oracle_mod
    b = W.with_prediction_noise(W.random_small(120, 92, n_max=25, M_lo=10, M_hi=60, a_max=20), eps)
    n_ev = 0
    for k in range(b.n_inst):
        req, M = b.instance(k)
        out = O.simulate(req, M, O.MCSF_PROT, alpha=(1, 10))
        n_ev += out["evictions"]
        if out["status"] == 0 and len(req):
            check_schedule(req, M, out)
    assert n_ev > 0


def test_protected_mcsf_unconstrained(oracle_mod):
    """Budget large enough for every projection and every realised batch: c = a + o."""
    O = oracle_mod
    b = W.with_prediction_noise(W.random_small(60, 93, n_max=12, M_lo=4, M_hi=30), 0.8)
    for k in range(b.n_inst):
        req, _ = b.instance(k)
        if len(req) == 0:
            continue
        M = int(2 * (req[:, 1] + np.maximum(req[:, 2], req[:, 3])).sum())
        out = O.simulate(req, M, O.MCSF_PROT, alpha=(1, 2))
        assert out["status"] == 0 and (out["completion"] == req[:, 0] + req[:, 2]).all()


# ----------------------------------------------------------------------------------------
# NEXT-4: wall clock under the affine batch time (DESIGN Q28)
# ----------------------------------------------------------------------------------------
def test_wallclock_closed_forms(oracle_mod):
    """A single request (s, o) arriving at 3: rounds 3..2+o, prefill s then o-1 decode tokens,
    so W(c) = o c0 + c1 (s + o - 1); with c0 = 1, c1 = 0 the wall clock is the round count."""
    O = oracle_mod
    for s, o in ((1, 1), (4, 7), (9, 2)):
        out = O.simulate([[3, s, o, o]], s + o, 0)
        w = O.wallclock([[3, s, o, o]], out["start"], out["completion"], 5, 2, 1, 64, 16)
        assert w["tel_wall"] == o * 5 + 2 * (s + o - 1) == w["makespan_wall"]
        assert w["bins"].sum() == s + o - 1                       # token conservation
        assert list(w["mem"][:o]) == [s + k for k in range(1, o + 1)]


def test_wallclock_unit_clock_is_tel(oracle_mod):
    """c0 = 1, c1 = 0 (one time unit per round) reproduces TEL and the makespan in rounds;
    the memory trace's maximum is the peak; bins conserve every processed token."""
    O = oracle_mod
    b = W.random_small(80, 95, n_max=20, M_lo=8, M_hi=50, a_max=15)
    for k in range(b.n_inst):
        req, M = b.instance(k)
        if len(req) == 0:
            continue
        out = O.simulate(req, M, 0)
        span = int(out["makespan"] - req[0, 0])
        w = O.wallclock(req, out["start"], out["completion"], 1, 0, 1, span + 1, span + 1)
        assert w["tel_wall"] == out["tel"] and w["makespan_wall"] == span
        assert w["mem"].max() == out["peak"]
        w2 = O.wallclock(req, out["start"], out["completion"], 3, 1, 7, 10_000, 0)
        assert w2["bins"].sum() == int((req[:, 1] + req[:, 2] - 1).sum())


# ----------------------------------------------------------------------------------------
# Round 2: eviction policies against hand-worked cases and an independent literal re-run
# ----------------------------------------------------------------------------------------
R2 = json.loads((GOLDEN / "round2_pins.json").read_text())
POL2 = dict(POL, mcsf_prot=4, mcsf_prot_raise=5)


@pytest.mark.parametrize("case", R2["cases"], ids=lambda c: c["name"])
def test_round2_worked_examples(oracle_mod, case):
    O = oracle_mod
    out = O.simulate(case["req"], case["M"], POL2[case["policy"]], alpha=tuple(case["alpha"]),
                     beta_thresh=case.get("beta_thresh", 0), seed=case.get("seed", 0),
                     gid=case.get("gid", 0))
    for k, v in case["expect"].items():
        got = list(out[k]) if isinstance(v, list) else out[k]
        assert got == v, (k, got, v)


def test_round2_beta_draws_are_philox(oracle_mod):
    """The draws written into the alpha-beta pin (computed with workloads' numpy Philox) are
    what the oracle's Philox gives on counter (t, pass, idx, 0) and key = seed halves (gid 0)."""
    case = next(c for c in R2["cases"] if c["policy"] == "alpha_beta")
    seed, t = case["seed"], case["draws"]["t"]
    for p, row in enumerate(case["draws"]["by_pass"]):
        for idx, hx in enumerate(row):
            got = oracle_mod.philox4x32_10([t, p, idx, 0], [seed & 0xFFFFFFFF, seed >> 32])[0]
            assert got == int(hx, 16)
            ref = W._philox_np([t], [p], [idx], [0], [seed & 0xFFFFFFFF], [seed >> 32])[0][0]
            assert int(ref) == int(hx, 16)


@pytest.mark.parametrize("case", R2["tel"], ids=lambda c: c["name"])
def test_or_tel_pins(oracle_mod, case):
    req = np.asarray(case["req"], np.int32).reshape(-1, 4)
    assert oracle_mod.tel(req, np.asarray(case["completion"], np.int32)) == case["tel"]


def test_alpha_beta_rejects_beta_zero_and_caps_passes(oracle_mod):
    """beta = 0 never clears (DESIGN Q29): refused.  A tiny beta (threshold 1 of 2^32) on the
    E9 overflow: 65536 passes evict nobody, so the run ends LIVELOCK at that overflow (t=24)."""
    O = oracle_mod
    e9 = [[0, 1, 40, 40], [0, 1, 40, 40]]
    with pytest.raises(ValueError):
        O.simulate(e9, 50, 3, alpha=(3, 10), beta_thresh=0)
    with pytest.raises(ValueError):
        O.simulate_batch([0, 2], e9, [50], 3, alpha=(3, 10), beta_thresh=0)
    with pytest.raises(ValueError):
        O.simulate(e9, 50, 3, alpha=(3, 10), beta_thresh=2**32 + 1)
    out = O.simulate(e9, 50, 3, alpha=(3, 10), beta_thresh=1, seed=3)
    assert out["status"] == 2 and out["evictions"] == 0 and out["decision_rounds"] == 1


def _literal_rerun(req, M, policy, alpha, cap):
    """An independent, literal re-run of alpha-greedy or protected MC-SF
     written from the paper's rules, with NO cycle detection: it stops only when
    every request has completed or at the round cap.  Returns (completion, finished)."""
    req = np.asarray(req, np.int64)
    n = len(req)
    a, s, o, op = (req[:, k] for k in range(4))
    B = ((alpha[1] - alpha[0]) * M) // alpha[1]
    p = [-1] * n
    c = [-1] * n
    R, S = [], []
    t, nxt = int(a[0]), 0
    while t <= cap:
        while nxt < n and a[nxt] <= t:
            R.append(nxt)
            nxt += 1
        S = [j for j in S if c[j] > t]
        if policy == 2:
            R.sort()
            L = sum(int(s[j]) + t + 1 - p[j] for j in S)
            while R and L + s[R[0]] + 1 <= B:
                i = R.pop(0)
                L += int(s[i]) + 1
                p[i], c[i] = t, t + int(o[i])
                S.append(i)
        else:
            R.sort(key=lambda i: (op[i], i))
            U = []
            for i in list(R):
                ok = True
                for tp in range(t + 1, t + max(int(op[k]) for k in U + [i]) + 1):
                    load = sum(int(s[j]) + tp - p[j] for j in S if op[j] >= tp - p[j])
                    load += sum(int(s[k]) + tp - t for k in U + [i] if op[k] >= tp - t)
                    if load > B:
                        ok = False
                        break
                if not ok:
                    break
                U.append(i)
            for i in U:
                R.remove(i)
                p[i], c[i] = t, t + int(o[i])
                S.append(i)
        if sum(int(s[j]) + t + 1 - p[j] for j in S) > M:
            for j in S:
                p[j] = c[j] = -1
                R.append(j)
            S = []
        if nxt == n and not R and not S:
            return c, True
        if not R and not S:
            t = int(a[nxt])
        else:
            t += 1
    return c, False


@pytest.mark.parametrize("policy", [2, 4])
def test_cycle_rule_matches_round_capped_rerun(oracle_mod, policy):
    """DESIGN Q24/Q25: declaring LIVELOCK early never changes a completion or the status
    against a literal run to the round cap (staggered arrivals, so cycles meet arrivals)."""
    O = oracle_mod
    b = W.random_small(400, 123 + policy, n_max=6, M_lo=6, M_hi=20, a_max=40)
    if policy == 4:
        b = W.with_prediction_noise(b, 0.8, seed=11)
    alpha = (1, 10) if policy == 2 else (0, 1)
    n_live = 0
    for k in range(b.n_inst):
        req, M = b.instance(k)
        if len(req) == 0:
            continue
        out = O.simulate(req, M, policy, alpha=alpha)
        if out["status"] == 1:
            continue
        cap = 16 * (int(req[-1, 0]) + int(req[:, 2].sum())) + 64
        comp, done = _literal_rerun(req, M, policy, alpha, cap)
        assert (out["status"] == 0) == done, (k, out["status"])
        # a request still in flight when the cap stops a run has not completed
        norm = lambda cs: [int(x) if x <= cap else -1 for x in cs]
        assert norm(out["completion"]) == norm(comp), k
        n_live += out["status"] == 2
    assert n_live > 0
