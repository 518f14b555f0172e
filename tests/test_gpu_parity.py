"""GPU parity: libkvsched.so (CUDA, through the C ABI) vs the CPU oracle, bit-exact.

Every field the ABI returns -- per-request completion and start rounds, per-instance TEL,
rounds, decision rounds, evictions, makespan, peak memory and status -- must equal the
oracle's on the same seeded inputs.  All integer: the bar is byte equality.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
KIND = {0: "mcsf", 1: "mcbench", 2: "alpha", 3: "alpha_beta", 4: "mcsf_protected", 5: "mcsf_protected_raise"}


@pytest.fixture(scope="module")
def K():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2502_07115_b200 as K
    from paper_2502_07115_b200 import build
    build.build()
    return K


@pytest.fixture(scope="module")
def ctx(K):
    c = K.Context(0)
    yield c
    c.close()


def oracle_run(O, b, pol, alpha=(0, 1), beta_thresh=0, seed=0, round_cap=0, gid0=0):
    return O.simulate_batch(b.offset, b.req, b.mem, pol, alpha=alpha, beta_thresh=beta_thresh,
                            seed=seed, round_cap=round_cap, gid0=gid0)


def gpu_run(K, ctx, b, pol, alpha=(0, 1), beta_thresh=0, seed=0, round_cap=0, id0=0, hints=None,
            flags=0):
    p = K.Policy(KIND[pol], alpha, beta_thresh, seed, round_cap, flags)
    return K.simulate(ctx, b, p, id0=id0, hints=hints if hints is not None else K.hints_of(b))


def assert_parity(o, g, b, label=""):
    fields = [("completion", "completion"), ("start", "start"), ("tel", "tel"), ("rounds", "rounds"),
              ("decision_rounds", "decision_rounds"), ("evictions", "evictions"),
              ("makespan", "makespan"), ("peak", "peak_mem"), ("status", "status")]
    for ok, gk in fields:
        x, y = np.asarray(o[ok]), np.asarray(g[gk])
        if not np.array_equal(x.astype(np.int64), y.astype(np.int64)):
            bad = np.nonzero(x != y)[0]
            i = int(bad[0])
            if ok in ("completion", "start"):
                k = int(np.searchsorted(b.offset, i, side="right") - 1)
            else:
                k = i
            raise AssertionError(f"{label}: {ok} differs at {len(bad)} positions; first {i} "
                                 f"(instance {k}): oracle {x[i]} gpu {y[i]}; "
                                 f"oracle status {o['status'][k]} gpu status {g['status'][k]}")


def check(K, ctx, O, b, pol, label, **kw):
    hints = kw.pop("hints", None)
    o = oracle_run(O, b, pol, **{k: v for k, v in kw.items() if k not in ("id0", "flags")},
                   gid0=kw.get("id0", 0))
    g = gpu_run(K, ctx, b, pol, hints=hints, **kw)
    assert_parity(o, g, b, label)
    return o, g


# ---------------------------------------------------------------------------------------
def test_library_loaded_is_in_tree(K):
    import paper_2502_07115_b200.kvsched as kv
    lib = K.load()
    assert Path(lib._name).resolve() == kv.LIB_PATH.resolve()


@pytest.mark.parametrize("case", json.loads((GOLDEN / "worked_examples.json").read_text())["cases"],
                         ids=lambda c: c["name"])
def test_worked_examples_on_gpu(K, ctx, oracle_mod, case):
    pol = {"mcsf": 0, "mcbench": 1, "alpha": 2, "alpha_beta": 3}[case["policy"]]
    b = W.from_instances([(case["req"], case["M"])])
    alpha = tuple(case.get("alpha", (0, 1)))
    o, g = check(K, ctx, oracle_mod, b, pol, case["name"], alpha=alpha)
    for k, v in case["expect"].items():
        gk = "peak_mem" if k == "peak" else k
        got = g[gk] if k in ("completion", "start") else g[gk][0]
        assert (list(got) == v) if isinstance(v, list) else (got == v), (k, got, v)


@pytest.mark.parametrize("pol", [0, 1])
@pytest.mark.parametrize("variant", ["a", "b"])
def test_c1_tiny(K, ctx, oracle_mod, pol, variant):
    b = W.c1(4000, 11, variant)
    check(K, ctx, oracle_mod, b, pol, f"C1{variant}")


@pytest.mark.parametrize("pol", [0, 1])
def test_c2_am1(K, ctx, oracle_mod, pol):
    b = W.am1(48, 12)
    check(K, ctx, oracle_mod, b, pol, "C2")


@pytest.mark.parametrize("pol", [0, 1])
def test_c5_am2(K, ctx, oracle_mod, pol):
    b = W.am2(6000, 13)
    check(K, ctx, oracle_mod, b, pol, "C5")


@pytest.mark.parametrize("maker", ["c5", "c2", "fuzz", "slow", "c1b", "cap"])
@pytest.mark.parametrize("pol", [0, 1])
def test_per_round_and_multi_round_modes(K, ctx, oracle_mod, maker, pol):
    """SCHED_FLAG_PER_ROUND (one Eq. 5 evaluation per round) and the default (a blocked head
    resolved over up to 64 rounds per warp pass) must both equal the oracle."""
    b = {"c5": lambda: W.am2(3000, 31), "c2": lambda: W.am1(16, 32),
         "fuzz": lambda: W.random_small(3000, 33, n_max=60, M_lo=4, M_hi=64, a_max=80),
         "slow": lambda: W.random_small(3000, 34, n_max=50, M_lo=8, M_hi=64, a_max=40, pred_slack=9),
         "c1b": lambda: W.c1(3000, 35, "b"),
         "cap": lambda: W.random_small(2000, 36, n_max=40, M_lo=6, M_hi=64, a_max=30)}[maker]()
    if maker == "slow" and pol == 1:
        return
    kw = dict(round_cap=23) if maker == "cap" else {}
    for flags in (0, 1):
        check(K, ctx, oracle_mod, b, pol, f"{maker} flags={flags}", flags=flags, **kw)


def _concat(*batches):
    insts = []
    for b in batches:
        insts += [b.instance(k) for k in range(b.n_inst)]
    return W.from_instances(insts)


@pytest.mark.parametrize("len_max", [12, 28, 48, 63])
@pytest.mark.parametrize("pol", [0, 1])
def test_lane_kernel_profile_widths(K, ctx, oracle_mod, pol, len_max):
    """k_mc_lane (one lane per instance) at every profile width it instantiates
    (max_len < 16, < 32, < 52, <= 63 -> 4, 8, 13, 16 words): equal to the oracle and to
    the one-warp-per-instance kernel (SCHED_FLAG_WARP_PER_INSTANCE)."""
    b = W.lane_mix(4000, 40 + len_max, len_max=len_max, gap_max=6)
    o, g = check(K, ctx, oracle_mod, b, pol, f"lane len_max={len_max}")
    w = gpu_run(K, ctx, b, pol, flags=K.kvsched.FLAG_WARP_PER_INSTANCE)
    assert_parity(o, w, b, "warp kernel")


@pytest.mark.parametrize("pol", [0, 1])
def test_lane_kernel_scope_edges(K, ctx, oracle_mod, pol):
    """A batch mixing instances inside the lane kernel's scope with every kind it hands to
    k_mc_small: n > 96, s > 7, arrival gaps > 511, o~ > o (MC-SF), invalid rows, empty
    instances, and n = 96 / s = 7 / gaps of 511 exactly at the edges."""
    inside = W.lane_mix(1500, 51, n_max=128, gap_max=8)
    big_n = W.lane_mix(60, 52, n_max=400, gap_max=3)
    big_s = W.lane_mix(300, 53, s_max=12, M_lo=20)
    gaps = W.lane_mix(300, 54, n_max=12, gap_max=900)
    edge = [([[0, 7, 57, 57]] * 96, 64), ([[0, 7, 57, 57]] * 97, 64), ([[0, 3, 5, 5]] * 128, 64),
            ([[0, 3, 5, 5]] * 129, 64), ([[0, 8, 5, 5]] * 110, 64), ([[0, 2, 5, 5]] * 100, 64),
            ([[0, 7, 1, 1], [511, 7, 1, 1], [1022, 1, 56, 56]], 64)]
    slow = [([[0, 2, 3, 9], [0, 1, 5, 5]], 20), ([[1, 3, 4, 4], [2, 2, 2, 6]], 12)]
    bad = [([[3, 1, 1, 1], [2, 1, 1, 1]], 10), ([[0, 1, 1, 1]] * 3, 6), ([], 7), ([[0, 5, 6, 6]], 10)]
    b = _concat(inside, big_n, W.from_instances(edge), big_s, gaps,
                W.from_instances(slow if pol == 0 else []), W.from_instances(bad))
    o, g = check(K, ctx, oracle_mod, b, pol, "lane scope edges")
    w = gpu_run(K, ctx, b, pol, flags=K.kvsched.FLAG_WARP_PER_INSTANCE)
    assert_parity(o, w, b, "warp kernel")
    h = gpu_run(K, ctx, b, pol, hints=(0, 0, 0))
    assert_parity(o, h, b, "measured hints")


@pytest.mark.parametrize("pol", [0, 1])
def test_flat_lane_kernel(K, ctx, oracle_mod, pol):
    """k_mc_flat: instances whose requests all arrive together (Arrival Model 1) and exceed
    the lane kernel's 96 positions run one per lane with the queue as a rank pointer; mixed
    with staggered large instances (k_mc_small), small ones (k_mc_lane) and invalid ones."""
    flat = [W.am1(40, 150 + pol, n=n, M=M) for n, M in ((97, 20), (500, 40), (1000, 64), (3000, 33))]
    paper = W.am1_paper(300, 151 + pol)                      # n 40-60 at t = 0: the lane kernel
    stag = W.lane_mix(40, 152 + pol, n_max=400, gap_max=3)    # n > 96, not simultaneous
    bad = W.from_instances([([[0, 9, 40, 40]] * 200, 40), ([[5, 1, 2, 2]] * 150 + [[4, 1, 2, 2]], 20)])
    b = _concat(*flat, paper, stag, bad)
    o, g = check(K, ctx, oracle_mod, b, pol, "flat lane kernel")
    w = gpu_run(K, ctx, b, pol, flags=K.kvsched.FLAG_WARP_PER_INSTANCE)
    assert_parity(o, w, b, "warp kernel")


@pytest.mark.parametrize("pol", [0, 1])
def test_small_kernel_large_queues(K, ctx, oracle_mod, pol):
    """More than 1024 requests per instance with M <= 64: the fused kernel keeps the waiting
    queue as a two-level shared-memory bitmap instead of one word per lane."""
    b = W.am1(6, 37, n=3000, M=48)
    for flags in (0, 1):
        check(K, ctx, oracle_mod, b, pol, f"n=3000 flags={flags}", flags=flags)
    c = W.random_small(60, 38, n_max=2500, M_lo=20, M_hi=64, a_max=3000)
    check(K, ctx, oracle_mod, c, pol, "ragged large n")


def test_am1_paper_draw(K, ctx, oracle_mod):
    b = W.am1_paper(400, 14)
    check(K, ctx, oracle_mod, b, 0, "AM1-paper")


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("pol", [0, 1, 2, 3])
@pytest.mark.parametrize("mhi", [64, 300])
def test_fuzz_ragged(K, ctx, oracle_mod, pol, mhi, flags):
    """Ragged batches (empty instances included), M up to 64 (fused kernel for MC) and up to
    300 (ring kernel), both evaluation modes."""
    b = W.random_small(3000, 15 + mhi, n_max=70, M_lo=4, M_hi=mhi, a_max=60)
    assert (b.sizes() == 0).any()
    kw = dict(alpha=(1, 10), beta_thresh=W.beta_threshold(0.3), seed=77) if pol >= 2 else {}
    check(K, ctx, oracle_mod, b, pol, f"fuzz M<={mhi}", flags=flags, **kw)


@pytest.mark.parametrize("pol", [0, 1])
def test_ring_kernel_on_small_budgets(K, ctx, oracle_mod, pol):
    """Force the shared-memory ring kernel (hint max_mem > 64) on small-M instances: both
    kernels must reproduce the oracle."""
    b = W.random_small(3000, 16, n_max=70, M_lo=4, M_hi=64, a_max=60)
    c = W.am2(2000, 17)
    for flags in (0, 1):
        check(K, ctx, oracle_mod, b, pol, "ring on small M", hints=(70, 65, 64), flags=flags)
        check(K, ctx, oracle_mod, c, pol, "ring on C5", hints=(c.max_requests(), 65, 64), flags=flags)


def test_prediction_overestimate_small(K, ctx, oracle_mod):
    """MC-SF with o~ >= o: early completions remove the unused projected tail."""
    b = W.random_small(3000, 18, n_max=50, M_lo=8, M_hi=64, a_max=40, pred_slack=8)
    assert (b.req[:, 3] > b.req[:, 2]).any()
    check(K, ctx, oracle_mod, b, 0, "o~ > o")


def _overestimate(b, eps, seed):
    """o~ = max(o, o^) with o^ the noisy prediction: MC-SF inputs with o~ >= o."""
    nb = W.with_prediction_noise(b, eps, seed=seed)
    req = nb.req.copy()
    req[:, 3] = np.maximum(req[:, 2], req[:, 3])
    return W.Batch(nb.offset.copy(), req, nb.mem.copy(), nb.name + "+over", dict(nb.meta))


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("shape", ["small", "long", "c4"])
def test_prediction_overestimate_ring(K, ctx, oracle_mod, shape, flags):
    """MC-SF with o~ >= o on the ring path (M > 64): k_ring lists the instances with early
    completions and k_prot runs them with alpha = 0 (the same schedule, see DESIGN Q10);
    instances with o~ = o stay on k_ring.  Includes k_prot's long-list overflow rerun."""
    b = {"small": lambda: W.random_small(2000, 60, n_max=40, M_lo=10, M_hi=80, a_max=30),
         "long": lambda: _long_batch(200, 61),
         "c4": lambda: W.c4(24, 62)}[shape]()
    b = _overestimate(b, 0.4, 63)
    if shape == "long":
        many = [([[0, 1, 2100, 2107]] * 40 + [[5, 3, 50, 50], [9, 2, 2500, 2500]], 200000),
                ([[0, 1, 3000, 3000]] * 33 + [[0, 1, 10, 12]] * 5, 120000)]
        b = _concat(b, W.from_instances(many))
    assert (b.req[:, 3] > b.req[:, 2]).any()
    ctx.reset_stats()
    ctx.set_timing(True)
    try:
        o, g = check(K, ctx, oracle_mod, b, 0, f"o~ > o on the ring path ({shape})", flags=flags)
        names = set(ctx.kernel_stats())
    finally:
        ctx.set_timing(False)
        ctx.reset_stats()
    assert "k_prot<MCSF,early>" in names and ("k_mc_ring<MCSF>" in names or "k_ring<MCSF>" in names), names
    assert (o["status"] == 0).sum() > 0


@pytest.mark.parametrize("name,pol,alpha,beta", W.C4_POLICIES, ids=[p[0] for p in W.C4_POLICIES])
def test_c4_policies(K, ctx, oracle_mod, name, pol, alpha, beta):
    b = W.c4(48, 19)
    polid = {"mcsf": 0, "mcbench": 1, "alpha": 2, "alpha_beta": 3}[pol]
    kw = dict(alpha=alpha or (0, 1), beta_thresh=W.beta_threshold(beta or 0.0), seed=2025)
    for flags in (0, 1):
        check(K, ctx, oracle_mod, b, polid, name, flags=flags, **kw)


def _long_batch(n_inst, seed, n_max=60, M_lo=3000, M_hi=9000, o_max=6000, a_max=400):
    """Instances whose requests often outlast the 2048-round ring window of k_ring."""
    g = np.random.default_rng(seed)
    insts = []
    for _ in range(n_inst):
        M = int(g.integers(M_lo, M_hi + 1))
        n = int(g.integers(0, n_max + 1))
        a = np.sort(g.integers(0, a_max + 1, n))
        s_ = g.integers(1, 60, n)
        o = np.minimum(g.integers(1, o_max + 1, n), M - s_)
        insts.append((np.stack([a, s_, o, o], 1).astype(np.int32), M))
    return W.from_instances(insts)


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("pol", [0, 1, 2, 3])
def test_ring_window_and_long_requests(K, ctx, oracle_mod, pol, flags):
    """Requests longer than the ring window go through the per-lane long list; an instance
    with more than 32 of them in flight is rerun by the full-ring launch."""
    b = _long_batch(400, 40 + pol)
    many = [([[0, 1, 2100, 2100]] * 40 + [[5, 3, 50, 50], [9, 2, 2500, 2500]], 200000),
            ([[0, 1, 3000, 3000]] * 33 + [[0, 1, 10, 10]] * 5, 120000)]
    c = W.from_instances(many)
    kw = dict(alpha=(1, 10), beta_thresh=W.beta_threshold(0.3), seed=3) if pol >= 2 else {}
    check(K, ctx, oracle_mod, b, pol, "long requests", flags=flags, **kw)
    check(K, ctx, oracle_mod, c, pol, "long-list overflow -> full ring", flags=flags, **kw)


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("eps", [0.2, 0.5, 0.8])
@pytest.mark.parametrize("shape", ["small", "long", "c4"])
def test_protected_mcsf(K, ctx, oracle_mod, eps, shape, flags):
    """NEXT-1: noisy predictions, budget (1-alpha)M, clearing on overflow; with
    the quiet-round jumps (flags 0) and round by round (SCHED_FLAG_PER_ROUND)."""
    b = {"small": lambda: W.random_small(2000, 50, n_max=40, M_lo=10, M_hi=80, a_max=30),
         "long": lambda: _long_batch(300, 51),
         "c4": lambda: W.c4(32, 52)}[shape]()
    b = W.with_prediction_noise(b, eps, seed=53)
    for alpha in ((1, 10), (0, 1), (3, 10)):
        o, g = check(K, ctx, oracle_mod, b, 4, f"protected eps={eps} alpha={alpha}", alpha=alpha,
                     flags=flags)
    if shape == "small":
        assert o["evictions"].sum() > 0


@pytest.mark.parametrize("pol", [2, 3])
def test_alpha_with_evictions(K, ctx, oracle_mod, pol):
    """Tight budgets force overflows, evictions and (for alpha-greedy) livelocks."""
    b = W.random_small(3000, 20, n_max=40, M_lo=10, M_hi=80, a_max=20)
    for alpha in ((1, 10), (0, 1), (3, 10)):
        for flags in (0, 1):
            o, g = check(K, ctx, oracle_mod, b, pol, f"alpha={alpha}", alpha=alpha,
                         beta_thresh=W.beta_threshold(0.25), seed=5, flags=flags)
    assert o["evictions"].sum() > 0
    assert (o["status"] == 2).any() or pol == 3


@pytest.mark.parametrize("lam", [0.4, 2.0])
@pytest.mark.parametrize("pol", [0, 1])
def test_c3_trace(K, ctx, oracle_mod, lam, pol):
    b = W.c3(2, 21, lam)
    for flags in (0, 1):
        check(K, ctx, oracle_mod, b, pol, f"C3 lam={lam}", flags=flags)


@pytest.mark.parametrize("pol", [0, 1, 2, 3])
def test_round_cap_livelock(K, ctx, oracle_mod, pol):
    """An explicit round cap stops runs mid-flight: both sides report LIVELOCK with the same
    partial counters and completions."""
    b = W.random_small(2000, 22, n_max=40, M_lo=6, M_hi=120, a_max=30)
    for cap, flags in ((5, 0), (17, 1), (40, 0), (40, 1), (61, 0)):
        kw = dict(round_cap=cap, flags=flags)
        if pol >= 2:
            kw.update(alpha=(1, 10), beta_thresh=W.beta_threshold(0.4), seed=3)
        o, _ = check(K, ctx, oracle_mod, b, pol, f"cap={cap}", **kw)
        assert (o["status"] == 2).any()


@pytest.mark.parametrize("pol", [0, 1, 2, 3])
def test_invalid_instances(K, ctx, oracle_mod, pol):
    insts = [([[0, 5, 6, 6]], 10), ([[3, 1, 1, 1], [2, 1, 1, 1]], 10), ([[0, 0, 1, 1]], 10),
             ([[0, 1, 3, 2]], 10), ([], 7), ([[0, 1, 1, 1]] * 3, 6), ([[0, 2, 3, 3], [1, 60, 3, 3]], 62),
             ([[0, 1, 2, 2], [0, 1, 2, 2], [0, 1, 5, 5]], 6)]
    b = W.from_instances(insts)
    check(K, ctx, oracle_mod, b, pol, "invalid", alpha=(1, 4), beta_thresh=2**31, seed=9)


def test_shard_invariance(K, ctx, oracle_mod):
    """Outputs do not depend on how the batch is split (instance_id0 keys the RNG)."""
    b = W.random_small(1500, 23, n_max=40, M_lo=10, M_hi=80, a_max=20)
    kw = dict(alpha=(1, 10), beta_thresh=W.beta_threshold(0.3), seed=11)
    whole = gpu_run(K, ctx, b, 3, **kw)
    cut = 611
    lo, hi = b.subset(range(cut)), b.subset(range(cut, b.n_inst))
    g0 = gpu_run(K, ctx, lo, 3, id0=0, **kw)
    g1 = gpu_run(K, ctx, hi, 3, id0=cut, **kw)
    for k in ("tel", "evictions", "status"):
        assert np.array_equal(whole[k], np.concatenate([g0[k], g1[k]]))
    assert np.array_equal(whole["completion"], np.concatenate([g0["completion"], g1["completion"]]))
    o1 = oracle_run(oracle_mod, hi, 3, gid0=cut, **kw)
    assert np.array_equal(o1["completion"], g1["completion"])


def test_unmeasured_hints(K, ctx, oracle_mod):
    """hints = 0 -> the library measures the bounds itself."""
    b = W.random_small(500, 24, n_max=50, M_lo=4, M_hi=200)
    o = oracle_run(oracle_mod, b, 0)
    g = gpu_run(K, ctx, b, 0, hints=(0, 0, 0))
    assert_parity(o, g, b, "measured hints")


def test_hint_violation_is_unsupported(K, ctx):
    b = W.random_small(200, 25, n_max=50, M_lo=20, M_hi=60)
    g = gpu_run(K, ctx, b, 0, hints=(20, 64, 63))
    big = b.sizes() > 20
    assert (g["status"][big] == 3).all() and (g["status"][~big] != 3).all()


def test_latency_kernel(K, ctx, oracle_mod):
    import torch
    b = W.am2(3000, 26)
    o = oracle_run(oracle_mod, b, 0)
    dev = torch.device("cuda", 0)
    off, req, _ = K.to_device(b, dev)
    comp = torch.from_numpy(o["completion"]).to(dev)
    tel = torch.empty(b.n_inst, dtype=torch.int64, device=dev)
    tot = torch.empty(1, dtype=torch.int64, device=dev)
    ctx.latency(off, req, comp, tel, tot)
    torch.cuda.synchronize()
    assert np.array_equal(tel.cpu().numpy(), o["tel"])
    assert int(tot.item()) == int(o["tel"].sum())
    comp[5] = -1
    ctx.latency(off, req, comp, tel, tot)
    torch.cuda.synchronize()
    k = int(np.searchsorted(b.offset, 5, side="right") - 1)
    assert tel[k].item() == -1


@pytest.mark.parametrize("pol", [0, 1, 2])
def test_maximum_sizes(K, ctx, oracle_mod, pol):
    """Instances at the build limits: 32768 requests (ring kernel), 16384 requests with
    M <= 64 (fused kernel, shared-memory queue), a request of length 32735 (SCHED_MAX_LEN)."""
    g = np.random.default_rng(80 + pol)
    n = 32768
    a = np.sort(g.integers(0, 20000, n))
    s_ = g.integers(1, 40, n)
    o = g.integers(1, 300, n)
    big = np.stack([a, s_, o, o], 1)
    n2 = 16384
    a2 = np.sort(g.integers(0, 3000, n2))
    s2 = g.integers(1, 6, n2)
    o2 = g.integers(1, 40, n2)
    small = np.stack([a2, s2, o2, o2], 1)
    longest = np.array([[0, 1, 32735, 32735], [5, 10, 100, 100], [7, 3, 20000, 20000]])
    b = W.from_instances([(big, 2000)])
    c = W.from_instances([(small, 48)])
    d = W.from_instances([(longest, 40000)])
    kw = dict(alpha=(1, 10)) if pol >= 2 else {}
    check(K, ctx, oracle_mod, b, pol, "n=32768", **kw)
    if pol < 2:
        check(K, ctx, oracle_mod, c, pol, "n=16384 small kernel", **kw)
    check(K, ctx, oracle_mod, d, pol, "length 32767", **kw)


def test_long_list_overflow_without_room_is_unsupported(K, ctx, oracle_mod):
    """k_prot keeps three rings per warp; a full-length rerun ring of 2^15 slots does not fit
    shared memory, so an instance with more than 32 long requests in flight is reported
    UNSUPPORTED (and only that one), never a wrong schedule."""
    many = ([[0, 1, 20000, 20000]] * 40, 2_000_000)
    fine = ([[0, 2, 30, 30], [3, 1, 20000, 20000]], 100_000)
    b = W.from_instances([fine, many, fine])
    g = gpu_run(K, ctx, b, 4, alpha=(1, 10))
    assert list(g["status"]) == [0, 3, 0]
    o = oracle_run(oracle_mod, b.subset([0, 2]), 4, alpha=(1, 10))
    assert list(o["tel"]) == [g["tel"][0], g["tel"][2]]
    lo, hi = int(b.offset[1]), int(b.offset[2])
    assert (g["completion"][lo:hi] == -1).all()


@pytest.mark.parametrize("n_inst,id0,seed", [(1, 0, 1), (3000, 0, 12345), (4097, 2**33 + 5, 7), (100000, 10**6, 99)])
def test_device_generation_matches_host_reference(K, ctx, oracle_mod, n_inst, id0, seed):
    """NEXT-3: sched_gen_am2 writes exactly the bytes of workloads.am2_counter; the
    generated batch then simulates to the oracle's schedules."""
    spec = W.Am2Spec(seed=seed)
    off, req, mem, n_req = ctx.gen_am2(n_inst, spec, id0=id0)
    import torch
    torch.cuda.synchronize()
    h = W.am2_counter(n_inst, spec, id0=id0)
    assert n_req == h.n_req
    assert np.array_equal(off.cpu().numpy(), h.offset)
    assert np.array_equal(req.cpu().numpy()[:n_req], h.req)
    assert np.array_equal(mem.cpu().numpy()[:n_inst], h.mem)
    if n_inst <= 4097:
        check(K, ctx, oracle_mod, h, 0, "generated batch")


def test_device_generation_edge_specs(K, ctx):
    """T_lo = T_hi = 0 (every instance empty) and a single-cell grid with a large lambda."""
    import torch
    for spec in (W.Am2Spec(T_lo=0, T_hi=0, seed=3), W.Am2Spec(lambdas=(6.0,), Ms=(64,), T_lo=1, T_hi=1024, s_lo=2, s_hi=9, seed=4)):
        off, req, mem, n_req = ctx.gen_am2(257, spec, id0=11)
        torch.cuda.synchronize()
        h = W.am2_counter(257, spec, id0=11)
        assert np.array_equal(off.cpu().numpy(), h.offset)
        assert np.array_equal(req.cpu().numpy()[:n_req], h.req[:n_req])


@pytest.mark.parametrize("maker", ["c5", "c4", "fuzz", "c3"])
def test_wallclock_kernel(K, ctx, oracle_mod, maker):
    """NEXT-4: sched_wallclock on GPU schedules equals the oracle's round-by-round clock."""
    import torch
    b = {"c5": lambda: W.am2(400, 61), "c4": lambda: W.c4(8, 62),
         "fuzz": lambda: W.random_small(300, 63, n_max=40, M_lo=6, M_hi=200, a_max=700),
         "c3": lambda: W.c3(1, 64, 2.0)}[maker]()
    dev = torch.device("cuda", 0)
    off, req, mem = K.to_device(b, dev)
    out = K.alloc_outputs(b.n_inst, b.n_req, dev)
    ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=K.hints_of(b))
    c0, c1, bw, nb, tl = 40, 3, 997, 64, 300
    w = ctx.wallclock(off, req, mem, out["start"], out["completion"], c0, c1, bw, nb, tl)
    torch.cuda.synchronize()
    st, cp = out["start"].cpu().numpy(), out["completion"].cpu().numpy()
    tw, mw = w["tel_wall"].cpu().numpy(), w["makespan_wall"].cpu().numpy()
    bins, memt = w["bins"].cpu().numpy(), w["mem"].cpu().numpy()
    for k in range(min(b.n_inst, 120)):
        r, M = b.instance(k)
        lo, hi = int(b.offset[k]), int(b.offset[k + 1])
        o = oracle_mod.wallclock(r, st[lo:hi], cp[lo:hi], c0, c1, bw, nb, tl)
        if len(r) == 0:
            assert tw[k] == 0 and mw[k] == 0
            continue
        assert (tw[k], mw[k]) == (o["tel_wall"], o["makespan_wall"]), k
        assert np.array_equal(bins[k], o["bins"]) and np.array_equal(memt[k], o["mem"]), k


@pytest.mark.parametrize("pol", [0, 2, 4])
def test_very_ragged_batch(K, ctx, oracle_mod, pol):
    """One 20000-request instance among 8000 tiny ones: the ring path sizes its scratch by the
    true row count (n_instances x max_requests would be ~3 GB)."""
    g = np.random.default_rng(85)
    big = np.stack([np.sort(g.integers(0, 9000, 20000)), g.integers(1, 30, 20000),
                    g.integers(1, 200, 20000), np.zeros(20000, np.int64)], 1)
    big[:, 3] = big[:, 2]
    small = W.random_small(8000, 86, n_max=6, M_lo=120, M_hi=300, a_max=10)
    insts = [(big, 3000)] + [small.instance(k) for k in range(small.n_inst)]
    b = W.from_instances(insts)
    kw = dict(alpha=(1, 10)) if pol >= 2 else {}
    o, g_ = check(K, ctx, oracle_mod, b, pol, "very ragged", **kw)
    assert (o["status"][1:] == g_["status"][1:]).all()


def test_lb_sorted_kernel(K, ctx, oracle_mod):
    """NEXT-2 (GPU part): the all-at-0 volume bound, bit-exact against the oracle's."""
    import torch
    batches = [W.c1(3000, 70, "a"), W.am1(64, 71), W.am1_paper(300, 72), W.am1(4, 73, n=5000, M=50),
               W.from_instances([([], 9), ([[3, 1, 2, 2], [3, 2, 1, 1]], 9), ([[0, 1, 2, 2], [1, 1, 2, 2]], 9)])]
    for b in batches:
        dev = torch.device("cuda", 0)
        off, req, mem = K.to_device(b, dev)
        lb = torch.empty(b.n_inst, dtype=torch.int64, device=dev)
        for hints in (K.hints_of(b), (0, 0, 0)):
            ctx.lb_sorted(off, req, mem, lb, hints=hints)
            torch.cuda.synchronize()
            got = lb.cpu().numpy()
            for k in range(b.n_inst):
                r, M = b.instance(k)
                if len(r) == 0:
                    want = 0
                elif (r[:, 0] != r[0, 0]).any():
                    want = -1
                else:
                    want = oracle_mod.lb_sorted(r, M)
                assert got[k] == want, (b.name, k, got[k], want)


def test_philox_known_answers_device(K, ctx):
    import torch
    ctr = torch.tensor([[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]],
                       dtype=torch.int64).to(torch.uint32).cuda()
    key = torch.tensor([[0, 0], [0xFFFFFFFF] * 2, [0xA4093822, 0x299F31D0]], dtype=torch.int64).to(torch.uint32).cuda()
    out = torch.zeros((3, 4), dtype=torch.uint32, device="cuda")
    ctx.philox(ctr, key, out)
    torch.cuda.synchronize()
    got = out.cpu().to(torch.int64).numpy().tolist()
    assert got[0] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert got[1] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert got[2] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def _host_outputs(b):
    outs = {"completion": np.empty(b.n_req, np.int32), "start": np.empty(b.n_req, np.int32)}
    for k in ("tel", "rounds", "decision_rounds", "evictions"):
        outs[k] = np.empty(b.n_inst, np.int64)
    for k in ("makespan", "peak_mem", "status"):
        outs[k] = np.empty(b.n_inst, np.int32)
    return outs


@pytest.mark.parametrize("pol", [0, 1, 2, 3, 4])
def test_host_path_pipelined_chunks(K, ctx, oracle_mod, pol, monkeypatch):
    """sched_run_instances_host cuts the batch into chunks (copy-in / kernel / copy-out on
    three streams); with tiny chunks every policy and both kernels must still match."""
    import paper_2502_07115_b200.kvsched as kv
    monkeypatch.setenv("KVSCHED_HOST_CHUNK_ROWS", "997")
    b = W.random_small(1500, 60 + pol, n_max=40, M_lo=6, M_hi=120, a_max=40)
    if pol == 4:
        b = W.with_prediction_noise(b, 0.3, seed=1)
    kw = dict(alpha=(1, 10), beta_thresh=W.beta_threshold(0.3), seed=4) if pol >= 2 else {}
    o = oracle_run(oracle_mod, b, pol, gid0=5, **kw)
    outs = _host_outputs(b)
    ctx.run_host(b.offset, b.req, b.mem, kv.Policy(KIND[pol], kw.get("alpha", (0, 1)), kw.get("beta_thresh", 0),
                                                   kw.get("seed", 0)), outs, id0=5, hints=K.hints_of(b))
    assert_parity(o, outs, b, "host chunks")
    outs0 = _host_outputs(b)        # hints measured on the host
    ctx.run_host(b.offset, b.req, b.mem, kv.Policy(KIND[pol], kw.get("alpha", (0, 1)), kw.get("beta_thresh", 0),
                                                   kw.get("seed", 0)), outs0, id0=5)
    assert_parity(o, outs0, b, "host chunks, measured hints")


@pytest.mark.parametrize("pol", [0, 1, 2, 4])
def test_packed_u16_rows(K, ctx, oracle_mod, pol, monkeypatch):
    """SCHED_REQ_U16X4_DELTA rows (half the bytes), decoded on the device, through both the
    device-pointer call and the chunked host path, give the same bytes as int32 rows."""
    import paper_2502_07115_b200.kvsched as kv
    b = W.random_small(1500, 90 + pol, n_max=50, M_lo=6, M_hi=120, a_max=300)
    if pol == 4:
        b = W.with_prediction_noise(b, 0.3, seed=2)
    kw = dict(alpha=(1, 10)) if pol >= 2 else {}
    o = oracle_run(oracle_mod, b, pol, **kw)
    p = K.Policy(KIND[pol], kw.get("alpha", (0, 1)))
    g = K.simulate(ctx, b, p, hints=K.hints_of(b), packed=True)
    assert_parity(o, g, b, "packed, device")
    monkeypatch.setenv("KVSCHED_HOST_CHUNK_ROWS", "1024")
    pk = b.packed_u16()
    outs = _host_outputs(b)
    ctx.run_host(b.offset, pk, b.mem, p, outs, hints=K.hints_of(b), req_format=kv.REQ_U16X4_DELTA)
    assert_parity(o, outs, b, "packed, host chunks")
    outs = _host_outputs(b)
    ctx.run_host(b.offset, pk, b.mem, p, outs, req_format=kv.REQ_U16X4_DELTA)      # host-measured hints
    assert_parity(o, outs, b, "packed, host, measured hints")


def _expected_latency16(o, b):
    c = np.asarray(o["completion"]).astype(np.int64)
    d = c - b.req[:, 0].astype(np.int64)
    return np.where((c < 0) | (d < 0) | (d > 65534), 65535, d).astype(np.uint16)


@pytest.mark.parametrize("fmt", ["u8", "p16"])
@pytest.mark.parametrize("pol", [0, 1, 2, 4])
def test_packed_rows_and_latency16(K, ctx, oracle_mod, pol, fmt, monkeypatch):
    """SCHED_REQ_U8X4_DELTA rows (a quarter of the int32 bytes), SCHED_REQ_P16 rows (an
    eighth; o~ = o) and the compact latency16 output (c_i - a_i as uint16; 65535 for
    unfinished requests): device-pointer call and chunked host path, with and without the
    int32 completion output beside it."""
    import paper_2502_07115_b200.kvsched as kv
    if fmt == "p16" and pol == 4:
        return                                    # P16 carries o~ = o only
    if fmt == "u8":
        b = W.random_small(1500, 120 + pol, n_max=50, M_lo=6, M_hi=120, a_max=200)
    else:
        b = W.lane_mix(1500, 130 + pol, len_max=63, s_max=8, gap_max=20)
    b = _concat(b, W.from_instances([([[0, 5, 6, 6]], 10), ([[0, 1, 1, 1], [0, 8, 2, 2]], 10)]))
    if pol == 4:
        b = W.with_prediction_noise(b, 0.3, seed=3)
    pk = b.packed_u8() if fmt == "u8" else b.packed_p16()
    assert pk is not None
    kw = dict(alpha=(1, 10)) if pol >= 2 else {}
    o = oracle_run(oracle_mod, b, pol, **kw)
    want = _expected_latency16(o, b)
    assert (want == 65535).any()
    p = K.Policy(KIND[pol], kw.get("alpha", (0, 1)))
    g = K.simulate(ctx, b, p, hints=K.hints_of(b), packed=fmt, latency16=True)
    assert_parity(o, g, b, f"{fmt} rows, device")
    assert np.array_equal(g["latency16"], want)
    g2 = K.simulate(ctx, b, p, hints=K.hints_of(b), packed=fmt, latency16=True, fields=("tel", "status"))
    assert np.array_equal(g2["latency16"], want)
    monkeypatch.setenv("KVSCHED_HOST_CHUNK_ROWS", "1000")
    rf = kv.REQ_U8X4_DELTA if fmt == "u8" else kv.REQ_P16
    for with_comp in (True, False):
        outs = _host_outputs(b)
        if not with_comp:
            del outs["completion"], outs["start"]
        outs["latency16"] = np.empty(b.n_req, np.uint16)
        ctx.run_host(b.offset, pk, b.mem, p, outs, hints=K.hints_of(b), req_format=rf)
        assert np.array_equal(outs["latency16"], want), with_comp
        if with_comp:
            assert_parity(o, outs, b, f"{fmt} rows, host chunks")
        else:
            assert np.array_equal(outs["tel"], np.asarray(o["tel"]))


@pytest.mark.parametrize("pol", [0, 1])
def test_host_path_lane_chunks(K, ctx, oracle_mod, pol, monkeypatch):
    """The host path on a lane-kernel batch cut into many chunks: four compute streams, each
    chunk's lane kernel on a quarter grid, size-scope fallbacks (n > 96) in every chunk."""
    import paper_2502_07115_b200.kvsched as kv
    monkeypatch.setenv("KVSCHED_HOST_CHUNK_ROWS", "4000")
    b = _concat(W.am2(3000, 140 + pol), W.lane_mix(200, 141 + pol, n_max=130, gap_max=3))
    o = oracle_run(oracle_mod, b, pol)
    outs = _host_outputs(b)
    outs["latency16"] = np.empty(b.n_req, np.uint16)
    ctx.run_host(b.offset, b.req, b.mem, K.Policy(KIND[pol]), outs, hints=K.hints_of(b))
    assert_parity(o, outs, b, "host lane chunks")
    assert np.array_equal(outs["latency16"], _expected_latency16(o, b))


@pytest.mark.parametrize("chunks", [1, 5, 16, 97])
@pytest.mark.parametrize("pol", [0, 1])
def test_host_path_streamed(K, ctx, oracle_mod, pol, chunks, monkeypatch):
    """The streamed host path (P16 rows, MC policies on the lane path): one persistent lane
    launch decodes the wire rows itself as the chunks land (flags set by stream memory
    operations), size-scope instances (n > 96) beside it on the side stream, row-scope ones
    (s = 8) after it, chunk k copied out once its instances are counted.  Every output, the
    latency16 conversion, and byte equality with the chunked pipeline (KVSCHED_HOST_STREAM=0)."""
    import paper_2502_07115_b200.kvsched as kv
    monkeypatch.setenv("KVSCHED_HOST_STREAM_CHUNKS", str(chunks))
    b = _concat(W.am2(2500, 150 + pol), W.lane_mix(400, 151 + pol, n_max=130, s_max=8, gap_max=30))
    b = _concat(b, W.from_instances([([[0, 5, 6, 6]], 10), ([[0, 1, 1, 1], [0, 8, 2, 2]], 10)]))
    pk = b.packed_p16()
    assert pk is not None
    o = oracle_run(oracle_mod, b, pol)
    want = _expected_latency16(o, b)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("KVSCHED_HOST_STREAM", mode)
        outs = _host_outputs(b)
        outs["latency16"] = np.empty(b.n_req, np.uint16)
        ctx.run_host(b.offset, pk, b.mem, K.Policy(KIND[pol]), outs, hints=K.hints_of(b), req_format=kv.REQ_P16)
        assert ("streamed" in ctx.last_kernel()) == (mode == "1"), ctx.last_kernel()
        assert_parity(o, outs, b, f"host streamed={mode}")
        assert np.array_equal(outs["latency16"], want), mode
        res[mode] = outs
        outs2 = {k: np.empty_like(v) for k, v in outs.items() if k not in ("completion", "start")}
        ctx.run_host(b.offset, pk, b.mem, K.Policy(KIND[pol]), outs2, hints=K.hints_of(b), req_format=kv.REQ_P16)
        assert np.array_equal(outs2["latency16"], want), mode
        assert np.array_equal(outs2["tel"], np.asarray(o["tel"])), mode
    for k in res["1"]:
        assert np.array_equal(res["1"][k], res["0"][k]), k


def test_host_path(K, ctx, oracle_mod):
    """sched_run_instances_host (host buffers, copies inside the call) gives the same bytes."""
    import paper_2502_07115_b200.kvsched as kv
    b = W.am2(2000, 27)
    o = oracle_run(oracle_mod, b, 0)
    outs = {"completion": np.empty(b.n_req, np.int32), "start": np.empty(b.n_req, np.int32)}
    for k in ("tel", "rounds", "decision_rounds", "evictions"):
        outs[k] = np.empty(b.n_inst, np.int64)
    for k in ("makespan", "peak_mem", "status"):
        outs[k] = np.empty(b.n_inst, np.int32)
    ctx.run_host(b.offset, b.req, b.mem, kv.Policy("mcsf"), outs, hints=K.hints_of(b))
    assert_parity(o, outs, b, "host path")


def test_full_size_c5_sampled(K, ctx, oracle_mod):
    """The bench configuration at full size (10^6 AM2 instances, one launch as bench.py
    times it); 300 sampled instances recomputed one by one by the oracle."""
    import torch
    b = W.am2(1_000_000, 5)
    dev = torch.device("cuda", 0)
    off, req, mem = K.to_device(b, dev)
    out = K.alloc_outputs(b.n_inst, b.n_req, dev)
    ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=K.hints_of(b))
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    assert (g["status"][:b.n_inst] == 0).all()
    ks = np.random.default_rng(0).choice(b.n_inst, 300, replace=False)
    ks[:2] = [0, b.n_inst - 1]
    for k in ks:
        req_k, M = b.instance(int(k))
        o = oracle_mod.simulate(req_k, M, 0)
        lo, hi = int(b.offset[k]), int(b.offset[k + 1])
        assert np.array_equal(o["completion"], g["completion"][lo:hi])
        assert o["tel"] == g["tel"][k] and o["rounds"] == g["rounds"][k]
        assert o["peak"] == g["peak_mem"][k] and o["decision_rounds"] == g["decision_rounds"][k]


@pytest.mark.parametrize("pol", [0, 1])
def test_full_size_c5_every_instance(K, ctx, oracle_mod, pol):
    """The bench configuration at full size (10^6 AM2 instances, 5 * 10^7 requests), every
    output of every instance against the oracle (the oracle runs on all host cores)."""
    b = W.am2(1_000_000, 5)
    g = gpu_run(K, ctx, b, pol)
    o = oracle_run(oracle_mod, b, pol)
    assert_parity(o, g, b, f"C5 full, policy {pol}")


@pytest.mark.parametrize("name,pol,alpha,beta", W.C4_POLICIES, ids=[p[0] for p in W.C4_POLICIES])
def test_c4_large_every_instance(K, ctx, oracle_mod, name, pol, alpha, beta):
    """C4 (trace-shaped, 1000 requests per instance) at 10^4 instances per Table-1 policy,
    every output of every instance against the oracle."""
    b = W.c4(10_000, 4)
    polid = {"mcsf": 0, "mcbench": 1, "alpha": 2, "alpha_beta": 3}[pol]
    kw = dict(alpha=alpha or (0, 1), beta_thresh=W.beta_threshold(beta or 0.0), seed=2025)
    check(K, ctx, oracle_mod, b, polid, f"C4 10^4 {name}", **kw)


@pytest.mark.parametrize("pol", [0, 1])
def test_full_size_c2_every_instance(K, ctx, oracle_mod, pol):
    """The bench's secondary configuration at full size (10^4 AM1 instances of 1000 requests
    at t = 0, M = 40; k_mc_flat), every output of every instance against the oracle."""
    b = W.am1(10_000, seed=2)
    g = gpu_run(K, ctx, b, pol)
    o = oracle_run(oracle_mod, b, pol)
    assert_parity(o, g, b, f"C2 full, policy {pol}")


# ---------------------------------------------------------------------------------------
# Round 2: the cycle rule only once nothing is left to arrive (DESIGN Q24/Q25), the beta
# pass cap and beta = 0 rejection (Q29), the hand-worked eviction cases
# ---------------------------------------------------------------------------------------
R2 = json.loads((GOLDEN / "round2_pins.json").read_text())


@pytest.mark.parametrize("case", R2["cases"], ids=lambda c: c["name"])
def test_round2_worked_examples_on_gpu(K, ctx, oracle_mod, case):
    pol = {"alpha": 2, "alpha_beta": 3, "mcsf_prot": 4, "mcsf_prot_raise": 5}[case["policy"]]
    b = W.from_instances([(case["req"], case["M"])])
    o, g = check(K, ctx, oracle_mod, b, pol, case["name"], alpha=tuple(case["alpha"]),
                 beta_thresh=case.get("beta_thresh", 0), seed=case.get("seed", 0),
                 id0=case.get("gid", 0))
    for k, v in case["expect"].items():
        gk = "peak_mem" if k == "peak" else k
        got = g[gk] if k in ("completion", "start") else g[gk][0]
        assert (list(got) == v) if isinstance(v, list) else (got == v), (k, got, v)


@pytest.mark.parametrize("pol", [2, 3, 4])
@pytest.mark.parametrize("flags", [0, 1])
def test_cycles_meeting_arrivals(K, ctx, oracle_mod, pol, flags):
    """Staggered arrivals into tight budgets: evictions cycle while requests are still to
    arrive, so the cycle rule must wait for the last arrival (both sides)."""
    b = W.random_small(4000, 130 + pol, n_max=12, M_lo=6, M_hi=40, a_max=80)
    kw = dict(alpha=(1, 10))
    if pol == 3:
        kw.update(beta_thresh=W.beta_threshold(0.2), seed=17)
    if pol == 4:
        b = W.with_prediction_noise(b, 0.8, seed=12)
        kw = dict(alpha=(0, 1))
    o, _ = check(K, ctx, oracle_mod, b, pol, f"cycles pol={pol}", flags=flags, **kw)
    assert o["evictions"].sum() > 0
    if pol != 3:
        assert (o["status"] == 2).any()


def test_alpha_beta_pass_cap_and_zero_beta(K, ctx, oracle_mod):
    """beta_thresh = 1: 65536 passes evict nobody at E9's overflow -> LIVELOCK on both sides;
    beta_thresh = 0 is refused by the ABI before anything is enqueued."""
    b = W.from_instances([([[0, 1, 40, 40], [0, 1, 40, 40]], 50), ([[0, 1, 3, 3]] * 3, 8)])
    o, g = check(K, ctx, oracle_mod, b, 3, "pass cap", alpha=(3, 10), beta_thresh=1, seed=3)
    assert list(g["status"]) == [2, 0]
    with pytest.raises(Exception):
        gpu_run(K, ctx, b, 3, alpha=(3, 10), beta_thresh=0)


@pytest.mark.parametrize("pol", [0, 1])
def test_zero_prediction_is_invalid_on_every_kernel(K, ctx, oracle_mod, pol):
    """o~ < 1 is INVALID for every policy (DESIGN Q8), whichever kernel picks the instance up:
    k_mc_lane (n <= 96), k_mc_flat (simultaneous, n > 96), k_mc_small, k_ring (M > 64)."""
    row0 = [0, 2, 3, 0]
    insts = [([row0, [0, 1, 3, 3]], 10),                                   # lane
             ([row0] + [[0, 1, 2, 2]] * 120, 40),                          # flat
             ([[0, 1, 2, 2]] * 100 + [[1, 1, 2, 0]], 40),                  # small
             ([row0, [3, 1, 3, 3]], 300),                                  # ring
             ([[0, 1, 3, 3], [0, 2, 4, 4]], 10)]                           # valid
    b = W.from_instances(insts)
    o, g = check(K, ctx, oracle_mod, b, pol, "o~ = 0")
    assert list(g["status"]) == [1, 1, 1, 1, 0]


@pytest.mark.parametrize("pol", [0, 1, 2, 4])
def test_hint_violation_does_not_spill_scratch(K, ctx, oracle_mod, pol):
    """An instance larger than the caller's max_requests hint comes first, so every later
    instance's rows lie past n_instances * hint.  The violator is UNSUPPORTED; later instances
    are either exact or UNSUPPORTED (their scratch rows would fall outside the allocation) --
    never written out of bounds (compute-sanitizer runs cover the same batch)."""
    big = ([[0, 1, 5, 5]] * 400, 300)
    rest = W.random_small(60, 27, n_max=15, M_lo=70, M_hi=200, a_max=20)
    insts = [big] + [rest.instance(k) for k in range(rest.n_inst)]
    b = W.from_instances(insts)
    kw = dict(alpha=(1, 10)) if pol >= 2 else {}
    g = gpu_run(K, ctx, b, pol, hints=(20, 300, 63), **kw)
    o = oracle_run(oracle_mod, b, pol, **kw)
    assert g["status"][0] == 3
    for k in range(1, b.n_inst):
        if g["status"][k] == 3:
            continue
        lo, hi = b.offset[k], b.offset[k + 1]
        assert g["status"][k] == o["status"][k] and g["tel"][k] == o["tel"][k], k
        assert np.array_equal(g["completion"][lo:hi], o["completion"][lo:hi]), k


@pytest.mark.parametrize("pol", [0, 1])
@pytest.mark.parametrize("big_n", [200, 700, 1500])
def test_hint_violation_any_prep_size(K, ctx, oracle_mod, pol, big_n):
    """An instance above the caller's max_requests hint is UNSUPPORTED whichever prep kernel
    its size would select (warp, 256-thread CTA, 1024-thread CTA): the launches are sized
    from the hint, so k_mc_prep_w takes every violator."""
    big = ([[0, 1, 5, 5]] * big_n, 300)
    rest = W.random_small(40, 28, n_max=15, M_lo=70, M_hi=200, a_max=20)
    b = W.from_instances([big] + [rest.instance(k) for k in range(rest.n_inst)] + [big])
    g = gpu_run(K, ctx, b, pol, hints=(20, 300, 63))
    o = oracle_run(oracle_mod, b, pol)
    assert g["status"][0] == 3 and g["status"][-1] == 3
    for k in range(1, b.n_inst - 1):
        if g["status"][k] == 3:
            continue
        lo, hi = b.offset[k], b.offset[k + 1]
        assert g["status"][k] == o["status"][k] and g["tel"][k] == o["tel"][k], k
        assert np.array_equal(g["completion"][lo:hi], o["completion"][lo:hi]), k


def test_lane_scope_far_arrivals(K, ctx, oracle_mod):
    """Arrival rounds near 2^30: the default cap min(2^30, ...) is reachable, so the lane and
    flat kernels must hand such instances to the general kernel."""
    base = 2**30 - 40
    insts = [([[base, 1, 30, 30], [base, 1, 30, 30]], 40),
             ([[base + 5, 2, 10, 10]] * 3, 30),
             ([[2**29 + 1, 1, 4, 4]], 10),
             ([[base, 1, 20, 20]] * 120, 41),
             ([[0, 1, 4, 4]], 10)]
    b = W.from_instances(insts)
    for pol in (0, 1):
        check(K, ctx, oracle_mod, b, pol, "far arrivals")


# ---------------------------------------------------------------------------------------
# Round 2: every-output parity at the configured sizes of C3 and C4 (BASELINE configs[2],
# configs[3])
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("lam", [0.4, 2.0])
@pytest.mark.parametrize("pol", [0, 1])
def test_c3_every_instance(K, ctx, oracle_mod, lam, pol):
    """C3 (trace-shaped, 10^4 requests per instance, M = 16492): 256 instances per lambda and
    MC policy, every output of every instance against the oracle."""
    b = W.c3(256, 300 + int(10 * lam), lam)
    check(K, ctx, oracle_mod, b, pol, f"C3 256 lam={lam}")


def test_c4_full_config_mcsf(K, ctx, oracle_mod):
    """C4 at the configured 10^5 instances (Table-1 regime, 1000 requests each), MC-SF, one
    launch, every output of every instance against the oracle."""
    b = W.c4(100_000, 4)
    check(K, ctx, oracle_mod, b, 0, "C4 10^5 MC-SF")


# ---------------------------------------------------------------------------------------
# DESIGN Q26b: protected MC-SF whose cleared requests re-enter with raised predictions
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("shape", ["small", "c4"])
@pytest.mark.parametrize("eps", [0.2, 0.8])
@pytest.mark.parametrize("flags", [0, 1])
def test_protected_raise(K, ctx, oracle_mod, shape, eps, flags):
    b = {"small": lambda: W.random_small(2000, 140, n_max=40, M_lo=10, M_hi=90, a_max=30),
         "c4": lambda: W.c4(48, 141)}[shape]()
    b = W.with_prediction_noise(b, eps, seed=13)
    o, g = check(K, ctx, oracle_mod, b, 5, f"Q26b {shape} eps={eps}", alpha=(1, 10), flags=flags)
    assert o["evictions"].sum() > 0
    assert (o["status"] == 0).sum() > 0
