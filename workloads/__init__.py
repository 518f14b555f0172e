"""workloads -- seeded synthetic instance generators (inputs only).

This module is the ONE thing the oracle tests and the CUDA path share: it draws
integer request tuples (a_i, s_i, o_i, o~_i) and budgets M with numpy's PCG64 and lays
them out in the CSR format both sides read.  It contains none of the scheduling method's
arithmetic (no admission, no memory projection, no latency).

Workload shapes (configs C1-C5 of BASELINE.json):
  C1  tiny: n=8, s~U{1..3}, o~U{1..8}, M=16; variant a: all a=0, b: a~U{0..5} sorted.
  C2  Arrival Model 1: n=1000 all at t=0, M=40, s~U{1..5}, o~U{1..M-s}.
  C3  trace-shaped online: per-round Poisson(lambda) arrivals, n=10^4,
      M=16492, lognormal lengths fitted to the published median/mean (DESIGN Q18,
      Q19), redrawn when s+o > M.
  C4  as C3 with n=1000, lambda=2.0 (the Table 1 regime).
  C5  Arrival Model 2: T~U{40..60}, Poisson(lambda) arrivals on rounds 1..T,
      s~U{1..5}, o~U{1..M-s}, on the grid lambda x M (DESIGN "Input recipe").
o~ = o everywhere (the paper's experiments use the true o).
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

GENERATOR_VERSION = "workloads-v1/numpy-%s/PCG64" % np.__version__

C5_LAMBDAS = (0.5, 0.75, 1.0, 1.25, 1.5)
C5_MS = (30, 35, 40, 45, 50)
TRACE_M = 16492
TRACE_S_MEDIAN, TRACE_S_MEAN = 11.0, 40.62
TRACE_O_MEDIAN, TRACE_O_MEAN = 45.0, 85.32
ROUNDS_PER_SECOND = 25.0             # DESIGN Q18 (assumption: ~40 ms per decode step)


@dataclass
class Batch:
    """CSR batch of independent instances.

    offset : int64 [n_inst+1]; requests of instance k are rows offset[k]:offset[k+1]
    req    : int32 [n_req, 4] rows {a, s, o, o~}, sorted by a within an instance
    mem    : int32 [n_inst] the KV budget M of each instance
    """
    offset: np.ndarray
    req: np.ndarray
    mem: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_inst(self) -> int:
        return int(self.mem.shape[0])

    @property
    def n_req(self) -> int:
        return int(self.req.shape[0])

    def sizes(self) -> np.ndarray:
        return np.diff(self.offset)

    def max_requests(self) -> int:
        return int(self.sizes().max()) if self.n_inst else 0

    def max_mem(self) -> int:
        return int(self.mem.max()) if self.n_inst else 0

    def max_len(self) -> int:
        return int(self.req[:, 2:4].max()) if self.n_req else 0

    def instance(self, k: int) -> tuple[np.ndarray, int]:
        lo, hi = int(self.offset[k]), int(self.offset[k + 1])
        return self.req[lo:hi], int(self.mem[k])

    def slice(self, lo: int, hi: int) -> "Batch":
        """Instances lo..hi-1 as a batch (contiguous: array views, no per-instance work)."""
        r0, r1 = int(self.offset[lo]), int(self.offset[hi])
        return Batch(self.offset[lo:hi + 1] - r0, self.req[r0:r1], self.mem[lo:hi],
                     self.name + "[slice]", dict(self.meta))

    def subset(self, ks) -> "Batch":
        ks = np.asarray(ks, dtype=np.int64)
        rows = [self.req[self.offset[k]:self.offset[k + 1]] for k in ks]
        sizes = np.array([r.shape[0] for r in rows], dtype=np.int64)
        off = np.zeros(len(ks) + 1, dtype=np.int64)
        np.cumsum(sizes, out=off[1:])
        req = np.concatenate(rows) if rows else np.zeros((0, 4), np.int32)
        return Batch(off, np.ascontiguousarray(req, dtype=np.int32),
                     np.ascontiguousarray(self.mem[ks]), self.name + "[subset]", dict(self.meta))

    def packed_u16(self):
        """Rows as uint16 {a_i - a_(i-1) (a_(-1) = 0 per instance), s, o, o~} (the C ABI's
        SCHED_REQ_U16X4_DELTA), or None if a value does not fit 16 bits."""
        if self.n_req == 0:
            return np.zeros((0, 4), np.uint16)
        a = self.req[:, 0].astype(np.int64)
        gap = np.diff(a, prepend=0)
        starts = self.offset[:-1][self.sizes() > 0]
        gap[starts] = a[starts]
        cols = np.stack([gap, self.req[:, 1], self.req[:, 2], self.req[:, 3]], 1)
        if cols.min() < 0 or cols.max() > 0xFFFF:
            return None
        return np.ascontiguousarray(cols.astype(np.uint16))

    def packed_u8(self):
        """Rows as uint8 {a_i - a_(i-1), s, o, o~} (SCHED_REQ_U8X4_DELTA), or None if a value
        does not fit a byte."""
        pk = self.packed_u16()
        if pk is None or (pk.size and pk.max() > 0xFF):
            return None
        return np.ascontiguousarray(pk.astype(np.uint8))

    def packed_p16(self):
        """Rows as uint16 {o-1:6 | s-1:3 | a_i - a_(i-1):7} with o~ = o (SCHED_REQ_P16), or
        None if the batch does not fit that encoding."""
        if self.n_req == 0:
            return np.zeros(0, np.uint16)
        pk = self.packed_u16()
        if pk is None:
            return None
        gap, s, o, op = (pk[:, j].astype(np.int64) for j in range(4))
        if (op != o).any() or o.min() < 1 or o.max() > 64 or s.min() < 1 or s.max() > 8 or gap.max() > 127:
            return None
        return np.ascontiguousarray(((o - 1) | ((s - 1) << 6) | (gap << 9)).astype(np.uint16))

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.offset, self.req, self.mem):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def from_instances(instances, name: str = "") -> Batch:
    """Batch from a list of (rows {a,s,o,o~}, M)."""
    rows = [np.asarray(r, dtype=np.int32).reshape(-1, 4) for r, _ in instances]
    sizes = np.array([r.shape[0] for r in rows], dtype=np.int64)
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    req = np.concatenate(rows) if rows else np.zeros((0, 4), np.int32)
    mem = np.array([m for _, m in instances], dtype=np.int32)
    return Batch(off, np.ascontiguousarray(req, dtype=np.int32), mem, name)


def _assemble(a, s, o, sizes, mem, name, meta) -> Batch:
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    req = np.empty((int(off[-1]), 4), dtype=np.int32)
    req[:, 0] = a
    req[:, 1] = s
    req[:, 2] = o
    req[:, 3] = o                         # o~ = o
    meta = dict(meta)
    meta["generator"] = GENERATOR_VERSION
    return Batch(off, req, np.ascontiguousarray(mem, dtype=np.int32), name, meta)


def _rng(seed) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def c1(n_inst: int, seed: int = 1, variant: str = "a") -> Batch:
    """C1: 8 requests, s~U{1..3}, o~U{1..8}, M=16; variant b staggers a~U{0..5}."""
    g = _rng([1, seed, 0 if variant == "a" else 1])
    n = 8
    s = g.integers(1, 4, size=(n_inst, n))
    o = g.integers(1, 9, size=(n_inst, n))
    if variant == "a":
        a = np.zeros((n_inst, n), dtype=np.int64)
    else:
        a = np.sort(g.integers(0, 6, size=(n_inst, n)), axis=1)
    sizes = np.full(n_inst, n, dtype=np.int64)
    return _assemble(a.ravel(), s.ravel(), o.ravel(), sizes, np.full(n_inst, 16), f"C1{variant}",
                     dict(seed=seed, variant=variant))


def am1(n_inst: int, seed: int = 2, n: int = 1000, M: int = 40) -> Batch:
    """C2 (Arrival Model 1): n requests at t=0, s~U{1..5}, o~U{1..M-s}."""
    g = _rng([2, seed, n, M])
    s = g.integers(1, 6, size=(n_inst, n))
    o = g.integers(1, M - s + 1)
    a = np.zeros_like(s)
    return _assemble(a.ravel(), s.ravel(), o.ravel(), np.full(n_inst, n, dtype=np.int64),
                     np.full(n_inst, M), "C2", dict(seed=seed, n=n, M=M))


def am1_paper(n_inst: int, seed: int = 20) -> Batch:
    """The paper's own AM1 draw: M~U{30..50}, n~U{40..60} per trial."""
    g = _rng([20, seed])
    M = g.integers(30, 51, size=n_inst)
    sizes = g.integers(40, 61, size=n_inst)
    Mrep = np.repeat(M, sizes)
    s = g.integers(1, 6, size=int(sizes.sum()))
    o = g.integers(1, Mrep - s + 1)
    return _assemble(np.zeros_like(s), s, o, sizes.astype(np.int64), M, "AM1-paper",
                     dict(seed=seed))


def am2_paper(n_inst: int, seed: int = 21) -> Batch:
    """The paper's own AM2 draw: per trial M~U{30..50}, T~U{40..60}, lambda~U[0.5, 1.5];
    Poisson(lambda) arrivals on each round 1..T (DESIGN Q20); s~U{1..5}; o~U{1..M-s}."""
    g = _rng([21, seed])
    M = g.integers(30, 51, size=n_inst)
    T = g.integers(40, 61, size=n_inst)
    lam = g.uniform(0.5, 1.5, size=n_inst)
    counts = g.poisson(lam[:, None], size=(n_inst, 60))
    counts[np.arange(60)[None, :] >= T[:, None]] = 0
    sizes = counts.sum(axis=1).astype(np.int64)
    rounds = np.broadcast_to(np.arange(1, 61, dtype=np.int64), (n_inst, 60))
    a = np.repeat(rounds.ravel(), counts.ravel())
    Mrep = np.repeat(M, sizes)
    s = g.integers(1, 6, size=a.shape[0])
    o = g.integers(1, Mrep - s + 1)
    return _assemble(a, s, o, sizes, M, "AM2-paper", dict(seed=seed))


def am2(n_inst: int, seed: int = 5, lambdas=C5_LAMBDAS, Ms=C5_MS, id0: int = 0) -> Batch:
    """C5 (Arrival Model 2): instance k sits on grid cell (k+id0) mod |grid| of
    lambda x M; T~U{40..60}; Poisson(lambda) arrivals on each round 1..T (DESIGN Q20);
    s~U{1..5}; o~U{1..M-s}."""
    g = _rng([5, seed, id0])
    grid = [(lam, m) for lam in lambdas for m in Ms]
    cell = (np.arange(n_inst, dtype=np.int64) + id0) % len(grid)
    lam = np.array([grid[c][0] for c in range(len(grid))])[cell]
    M = np.array([grid[c][1] for c in range(len(grid))], dtype=np.int64)[cell]
    T = g.integers(40, 61, size=n_inst)
    counts = g.poisson(lam[:, None], size=(n_inst, 60))
    counts[np.arange(60)[None, :] >= T[:, None]] = 0          # rounds 1..T only
    sizes = counts.sum(axis=1).astype(np.int64)
    rounds = np.broadcast_to(np.arange(1, 61, dtype=np.int64), (n_inst, 60))
    a = np.repeat(rounds.ravel(), counts.ravel())             # row-major: sorted per instance
    Mrep = np.repeat(M, sizes)
    s = g.integers(1, 6, size=a.shape[0])
    o = g.integers(1, Mrep - s + 1)
    return _assemble(a, s, o, sizes, M, "C5",
                     dict(seed=seed, id0=id0, lambdas=list(lambdas), Ms=list(Ms)))


def _lognormal_int(g, median, mean, size):
    mu = math.log(median)
    sigma = math.sqrt(2.0 * math.log(mean / median))          # DESIGN Q19
    x = np.exp(mu + sigma * g.standard_normal(size))
    return np.maximum(1, np.floor(x + 0.5)).astype(np.int64)


def trace_shaped(n_inst: int, seed: int = 3, n: int = 10_000, lam_round: float = 2.0,
                 M: int = TRACE_M) -> Batch:
    """C3/C4: per-round Poisson(lam_round) arrivals from round 0 until n
    requests arrived; s, o discretised lognormals fitted to the trace's median/mean
    (P:453), pair redrawn while s+o > M."""
    g = _rng([3, seed, n, int(round(lam_round * 1000)), M])
    n_rounds = int(math.ceil(n / lam_round * 1.3 + 64))
    counts = g.poisson(lam_round, size=(n_inst, n_rounds))
    csum = counts.cumsum(axis=1)
    while (csum[:, -1] < n).any():                            # extend (rare)
        extra = g.poisson(lam_round, size=(n_inst, n_rounds))
        counts = np.concatenate([counts, extra], axis=1)
        csum = counts.cumsum(axis=1)
        n_rounds = counts.shape[1]
    # arrival round of the j-th request = number of rounds whose cumulative count <= j
    j = np.arange(n, dtype=np.int64)
    a = np.stack([np.searchsorted(csum[k], j, side="right") for k in range(n_inst)])
    total = n_inst * n
    s = _lognormal_int(g, TRACE_S_MEDIAN, TRACE_S_MEAN, total)
    o = _lognormal_int(g, TRACE_O_MEDIAN, TRACE_O_MEAN, total)
    bad = s + o > M
    while bad.any():
        k = int(bad.sum())
        s[bad] = _lognormal_int(g, TRACE_S_MEDIAN, TRACE_S_MEAN, k)
        o[bad] = _lognormal_int(g, TRACE_O_MEDIAN, TRACE_O_MEAN, k)
        bad = s + o > M
    return _assemble(a.ravel(), s, o, np.full(n_inst, n, dtype=np.int64), np.full(n_inst, M),
                     "C3" if n == 10_000 else "C4",
                     dict(seed=seed, n=n, lam_round=lam_round, M=M))


def c3(n_inst: int, seed: int = 3, lam_round: float = 2.0) -> Batch:
    return trace_shaped(n_inst, seed, n=10_000, lam_round=lam_round)


def c4(n_inst: int, seed: int = 4) -> Batch:
    return trace_shaped(n_inst, seed, n=1000, lam_round=2.0)


# Table 1 rows as C-ABI policy parameters: (name, policy, alpha, beta)
C4_POLICIES = (
    ("MC-SF", "mcsf", None, None),
    ("MC-Benchmark", "mcbench", None, None),
    ("alpha=0.3", "alpha", (3, 10), None),
    ("alpha=0.25", "alpha", (1, 4), None),
    ("alpha=0.2,beta=0.2", "alpha_beta", (1, 5), 0.2),
    ("alpha=0.2,beta=0.1", "alpha_beta", (1, 5), 0.1),
    ("alpha=0.1,beta=0.2", "alpha_beta", (1, 10), 0.2),
    ("alpha=0.1,beta=0.1", "alpha_beta", (1, 10), 0.1),
)


def beta_threshold(beta: float) -> int:
    """beta in [0,1] -> integer threshold in [0, 2^32] (evict iff u32 < threshold)."""
    return int(round(beta * 2.0 ** 32))


def random_small(n_inst: int, seed: int, n_max: int = 40, M_lo: int = 4, M_hi: int = 64,
                 a_max: int = 30, len_max: int | None = None, pred_slack: int = 0) -> Batch:
    """Ragged fuzz batch for parity tests: n~U{0..n_max} (empty instances included),
    M~U{M_lo..M_hi}, s~U{1..M/4}, o~U{1..M-s} (capped by len_max), arrivals U{0..a_max}
    sorted.  pred_slack>0 draws o~ = o + U{0..pred_slack} (clipped to M-s)."""
    g = _rng([9, seed, n_max, M_lo, M_hi, a_max, pred_slack])
    sizes = g.integers(0, n_max + 1, size=n_inst).astype(np.int64)
    M = g.integers(M_lo, M_hi + 1, size=n_inst)
    Mrep = np.repeat(M, sizes)
    s = g.integers(1, np.maximum(2, Mrep // 4 + 1))
    hi = Mrep - s
    if len_max is not None:
        hi = np.minimum(hi, len_max)
    o = g.integers(1, np.maximum(hi, 1) + 1)
    a = g.integers(0, a_max + 1, size=int(sizes.sum()))
    # sort arrivals within each instance
    inst = np.repeat(np.arange(n_inst), sizes)
    order = np.lexsort((a, inst))
    a = a[order]
    b = _assemble(a, s, o, sizes, M, "fuzz", dict(seed=seed))
    if pred_slack > 0:
        extra = g.integers(0, pred_slack + 1, size=b.n_req)
        op = np.minimum(b.req[:, 2] + extra, np.repeat(M, sizes) - b.req[:, 1])
        b.req[:, 3] = np.maximum(op, b.req[:, 2])
    return b


def lane_mix(n_inst: int, seed: int, len_max: int = 63, n_max: int = 128, s_max: int = 7,
             gap_max: int = 40, M_lo: int = 8, M_hi: int = 64) -> Batch:
    """Parity batch shaped for the one-lane-per-instance MC kernel's scope edges:
    n~U{1..n_max}, M~U{M_lo..M_hi}, s~U{1..min(s_max, M-1)}, o~U{1..min(M-s, len_max)},
    arrival gaps U{0..gap_max} (o~ = o).  Choosing n_max > 128, s_max > 7 or gap_max > 511
    puts some instances outside that scope."""
    g = _rng([17, seed, len_max, n_max, s_max, gap_max, M_lo, M_hi])
    sizes = g.integers(1, n_max + 1, size=n_inst).astype(np.int64)
    M = g.integers(M_lo, M_hi + 1, size=n_inst)
    Mrep = np.repeat(M, sizes)
    s = g.integers(1, np.minimum(s_max, Mrep - 1) + 1)
    o = g.integers(1, np.minimum(Mrep - s, len_max) + 1)
    gaps = g.integers(0, gap_max + 1, size=int(sizes.sum()))
    starts = np.zeros(n_inst + 1, dtype=np.int64)
    np.cumsum(sizes, out=starts[1:])
    a = np.cumsum(gaps)
    a = a - np.repeat(a[starts[:-1]], sizes) + np.repeat(g.integers(0, 50, size=n_inst), sizes)
    return _assemble(a, s, o, sizes, M, "lane-mix", dict(seed=seed, len_max=len_max))


def with_prediction_noise(b: Batch, eps: float, seed: int = 7) -> Batch:
    """Replace o~ by a noisy prediction o^ ~ U((1-eps)o, (1+eps)o), rounded to
    an integer >= 1 on the host (DESIGN Q26): o^ = max(1, floor(o (1 + eps (2u - 1)) + 0.5)).
    Predictions may under- or over-shoot o; they are capped at 32735 (the build's length limit)."""
    g = _rng([13, seed, int(round(eps * 1000))])
    u = g.random(b.n_req)
    o = b.req[:, 2].astype(np.float64)
    pred = np.maximum(1, np.floor(o * (1.0 + eps * (2.0 * u - 1.0)) + 0.5)).astype(np.int64)
    req = b.req.copy()
    req[:, 3] = np.minimum(pred, 32735)
    meta = dict(b.meta)
    meta["prediction_noise_eps"] = eps
    return Batch(b.offset.copy(), req, b.mem.copy(), b.name + f"+noise{eps}", meta)


# ---------------------------------------------------------------------------------------
# NEXT-3: the AM2-grid generator as an integer counter-based spec (host reference).
# The CUDA path implements the same spec in sched_gen_am2_{count,fill}; both consume the same
# Poisson inversion tables (computed here, passed as inputs) so no floating point is involved
# in either generator.
#
#   instance g (global id), cell = g mod (|lambdas| |Ms|), lambda = lambdas[cell // |Ms|],
#   M = Ms[cell % |Ms|];  u(stream, j) = Philox4x32-10(counter (lo32 g, hi32 g, stream, j),
#   key (lo32 seed, hi32 seed));  mulhi(u, r) = (u * r) >> 32
#   T     = T_lo + mulhi(u(0, 0).x, T_hi - T_lo + 1)
#   count(r) for rounds r = 1..T: smallest c with u(1, r).x < cdf[lambda][c]  (c <= 31)
#   requests i = 0.. in arrival order: w = u(2, i); s = s_lo + mulhi(w.x, s_hi - s_lo + 1);
#   o = 1 + mulhi(w.y, M - s); o~ = o
# ---------------------------------------------------------------------------------------
GEN_AM2_VERSION = "am2-grid-v1"
POISSON_TABLE_LEN = 32


def _philox_np(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 (Salmon et al., SC'11) on uint32 numpy arrays."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32).copy() for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32).copy()
    k1 = np.asarray(k1, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = c0.astype(np.uint64) * M0
            p1 = c2.astype(np.uint64) * M1
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), p0.astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), p1.astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = k0 + W0
            k1 = k1 + W1
    return c0, c1, c2, c3


def _mulhi(u, r):
    return ((np.asarray(u, dtype=np.uint64) * np.asarray(r, dtype=np.uint64)) >> np.uint64(32)).astype(np.int64)


def poisson_cdf_table(lam: float) -> np.ndarray:
    """uint64 thresholds floor(P(X <= c) 2^32), c = 0..31, last one forced to 2^32."""
    p = math.exp(-lam)
    acc, out = 0.0, []
    for c in range(POISSON_TABLE_LEN):
        acc += p
        out.append(min(int(acc * 2.0 ** 32), 2 ** 32))
        p *= lam / (c + 1)
    out[-1] = 2 ** 32
    return np.array(out, dtype=np.uint64)


@dataclass
class Am2Spec:
    lambdas: tuple = C5_LAMBDAS
    Ms: tuple = C5_MS
    T_lo: int = 40
    T_hi: int = 60
    s_lo: int = 1
    s_hi: int = 5
    seed: int = 12345

    def tables(self) -> np.ndarray:
        return np.stack([poisson_cdf_table(l) for l in self.lambdas])


def am2_counter(n_inst: int, spec: Am2Spec = Am2Spec(), id0: int = 0) -> Batch:
    """Host reference of the counter-based AM2-grid generator (the spec above)."""
    g = np.arange(id0, id0 + n_inst, dtype=np.uint64)
    glo, ghi = (g & np.uint64(0xFFFFFFFF)).astype(np.uint32), (g >> np.uint64(32)).astype(np.uint32)
    k0 = np.full(n_inst, spec.seed & 0xFFFFFFFF, dtype=np.uint32)
    k1 = np.full(n_inst, (spec.seed >> 32) & 0xFFFFFFFF, dtype=np.uint32)
    ncell = len(spec.lambdas) * len(spec.Ms)
    cell = (g % np.uint64(ncell)).astype(np.int64)
    li, mi = cell // len(spec.Ms), cell % len(spec.Ms)
    M = np.asarray(spec.Ms, dtype=np.int64)[mi]
    cdf = spec.tables()
    z = np.zeros(n_inst, dtype=np.uint32)
    T = spec.T_lo + _mulhi(_philox_np(glo, ghi, z, z, k0, k1)[0], spec.T_hi - spec.T_lo + 1)
    counts = np.zeros((n_inst, spec.T_hi), dtype=np.int64)
    for r in range(1, spec.T_hi + 1):
        u = _philox_np(glo, ghi, np.full(n_inst, 1, np.uint32), np.full(n_inst, r, np.uint32), k0, k1)[0]
        c = (u.astype(np.uint64)[:, None] >= cdf[li]).sum(axis=1)      # smallest c with u < cdf[c]
        counts[:, r - 1] = np.where(r <= T, c, 0)
    sizes = counts.sum(axis=1)
    rounds = np.broadcast_to(np.arange(1, spec.T_hi + 1, dtype=np.int64), counts.shape)
    a = np.repeat(rounds.ravel(), counts.ravel())
    inst = np.repeat(np.arange(n_inst), sizes)
    start = np.zeros(n_inst + 1, dtype=np.int64)
    np.cumsum(sizes, out=start[1:])
    i = np.arange(a.shape[0], dtype=np.int64) - start[inst]
    gg = g[inst]
    w = _philox_np((gg & np.uint64(0xFFFFFFFF)).astype(np.uint32), (gg >> np.uint64(32)).astype(np.uint32),
                   np.full(a.shape[0], 2, np.uint32), i.astype(np.uint32), k0[inst], k1[inst])
    s = spec.s_lo + _mulhi(w[0], spec.s_hi - spec.s_lo + 1)
    o = 1 + _mulhi(w[1], np.maximum(M[inst] - s, 0))
    b = _assemble(a, s, o, sizes, M, "C5-counter", dict(spec=GEN_AM2_VERSION, seed=spec.seed, id0=id0))
    return b
