"""The seeded input generators (workloads/): determinism, shapes, ranges, moments."""
import math

import numpy as np

import workloads as W


def _check_batch(b):
    assert b.offset[0] == 0 and b.offset[-1] == b.n_req
    assert (np.diff(b.offset) >= 0).all()
    assert b.req.dtype == np.int32 and b.req.flags.c_contiguous
    for k in range(min(b.n_inst, 50)):
        req, M = b.instance(k)
        if len(req):
            assert (np.diff(req[:, 0]) >= 0).all()
            assert (req[:, 1] >= 1).all() and (req[:, 2] >= 1).all()
            assert (req[:, 1] + req[:, 3] <= M).all()


def test_deterministic():
    for f in (lambda: W.c1(10, 3, "b"), lambda: W.am1(3, 4), lambda: W.am2(100, 5),
              lambda: W.c4(2, 6)):
        assert f().sha256() == f().sha256()
    assert W.am2(100, 5).sha256() != W.am2(100, 6).sha256()


def test_shapes_and_ranges():
    for b in (W.c1(20, 1, "a"), W.c1(20, 1, "b"), W.am1(4, 2), W.am2(500, 3), W.c4(2, 4),
              W.random_small(50, 5), W.am1_paper(5, 6)):
        _check_batch(b)
    b = W.am2(2500, 7)
    assert set(np.unique(b.mem)) == set(W.C5_MS)
    assert b.req[:, 0].min() >= 1 and b.req[:, 0].max() <= 60      # rounds 1..T
    assert b.req[:, 1].max() <= 5
    b = W.am1(2, 2)
    assert (b.req[:, 0] == 0).all() and b.max_requests() == 1000 and (b.mem == 40).all()


def test_trace_moments():
    """Lognormal fit to the published medians/means: the medians are exact by
    construction; the means come out near 40.62 / 85.32 (truncation by s+o <= M)."""
    b = W.c3(2, 3)
    s, o = b.req[:, 1], b.req[:, 2]
    assert abs(np.median(s) - 11) <= 1 and abs(np.median(o) - 45) <= 2
    assert abs(s.mean() - 40.62) / 40.62 < 0.15 and abs(o.mean() - 85.32) / 85.32 < 0.1
    assert (b.mem == 16492).all() and b.max_requests() == 10_000
    # Poisson(2) per round -> about n/2 rounds of arrivals
    span = b.instance(0)[0][-1, 0]
    assert abs(span - 5000) < 400
    assert abs(math.sqrt(2 * math.log(40.62 / 11)) - 1.616) < 1e-3


def test_counter_generator_spec():
    """NEXT-3 host reference (workloads.am2_counter): deterministic, on the grid, ranges of
    P:408 (T in [40, 60], arrivals on rounds 1..T, s in [1, 5], o in [1, M - s]), Poisson
    counts with the right mean, Philox matching the published known-answer vector."""
    c = W._philox_np(np.array([0x243F6A88], np.uint32), np.array([0x85A308D3], np.uint32),
                     np.array([0x13198A2E], np.uint32), np.array([0x03707344], np.uint32),
                     np.array([0xA4093822], np.uint32), np.array([0x299F31D0], np.uint32))
    assert [int(x[0]) for x in c] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]
    t = W.poisson_cdf_table(1.0)
    assert (np.diff(t.astype(np.int64)) >= 0).all() and t[-1] == 2 ** 32
    assert abs(int(t[0]) / 2 ** 32 - math.exp(-1.0)) < 1e-9
    spec = W.Am2Spec()
    b = W.am2_counter(5000, spec, id0=123)
    assert b.sha256() == W.am2_counter(5000, spec, id0=123).sha256()
    _check_batch(b)
    assert b.req[:, 0].min() >= 1 and b.req[:, 0].max() <= 60
    assert b.req[:, 1].min() >= 1 and b.req[:, 1].max() <= 5
    cells = (np.arange(123, 5123) % 25)
    assert (b.mem == np.array(W.C5_MS)[cells % 5]).all()
    lam = np.array(W.C5_LAMBDAS)[cells // 5]
    assert abs(b.sizes().mean() / (lam * 50).mean() - 1) < 0.02
    # shards of the global id range concatenate to the whole
    x, y = W.am2_counter(2000, spec, id0=123), W.am2_counter(3000, spec, id0=2123)
    assert np.array_equal(np.concatenate([x.req, y.req]), b.req)


def test_packed_formats_roundtrip_and_slice():
    """The wire encodings decode back to the int32 rows (host-side check of the formats the
    C ABI accepts), and contiguous slices equal index subsets."""
    b = W.am2(3000, 7)
    for pk, width in ((b.packed_u16(), 16), (b.packed_u8(), 8)):
        assert pk is not None
        a = np.zeros(b.n_req, np.int64)
        for k in range(b.n_inst):
            lo, hi = int(b.offset[k]), int(b.offset[k + 1])
            a[lo:hi] = np.cumsum(pk[lo:hi, 0].astype(np.int64))
        assert np.array_equal(a, b.req[:, 0]) and np.array_equal(pk[:, 1:].astype(np.int32), b.req[:, 1:])
    p16 = b.packed_p16().astype(np.int64)
    assert np.array_equal((p16 & 63) + 1, b.req[:, 2]) and np.array_equal(((p16 >> 6) & 7) + 1, b.req[:, 1])
    gaps = p16 >> 9
    assert np.array_equal(gaps, b.packed_u16()[:, 0].astype(np.int64))
    assert W.with_prediction_noise(b, 0.3).packed_p16() is None        # o~ != o does not fit P16
    s = b.slice(100, 250)
    t = b.subset(range(100, 250))
    assert np.array_equal(s.offset, t.offset) and np.array_equal(s.req, t.req) and np.array_equal(s.mem, t.mem)
