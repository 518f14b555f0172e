"""oracle -- TEST INFRASTRUCTURE ONLY.

Python view of ``oracle/oracle.c``: a plain, slow, literal CPU transcription of
arXiv 2502.07115 (Algorithm 1 MC-SF, Algorithm 2 MC-Benchmark, the alpha-protection
baselines, the hindsight IP optimum on tiny instances).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  It shares no code with ``paper_2502_07115_b200`` (the
product path) and never imports it; the product path never imports it either.

Citations: ``P:<line>`` = line of PAPER.md (the paper's LaTeX source); ``DESIGN Qn`` =
the reading recorded in DESIGN.md where the paper is silent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "oracle.c"
_LIB = _HERE / "liboracle.so"

# policy ids of the oracle (its own numbering)
MCSF, MCBENCH, ALPHA, ALPHA_BETA, MCSF_PROT, MCSF_PROT_RAISE = 0, 1, 2, 3, 4, 5
# instance status
OK, INVALID, LIVELOCK = 0, 1, 2


def build(force: bool = False) -> Path:
    """Compile oracle.c with gcc (plain C11, -O2)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-Wall", "-shared", "-fPIC",
                               "-o", str(tmp), str(_SRC), "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        P = ctypes.c_void_p
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.or_philox4x32_10.argtypes = [P, P, P]
        L.or_projected_occupancy.argtypes = [i64, i64, i64, P, P, P, i64, P, P]
        L.or_projected_occupancy.restype = i64
        L.or_is_feasible.argtypes = [i64, i64, i64, P, P, P, i64, P, P]
        L.or_is_feasible.restype = ctypes.c_int
        L.or_simulate.argtypes = [i64, P, i32, i32, i32, i32, u64, u64, i64, u64, P, P, P]
        L.or_simulate.restype = ctypes.c_int
        L.or_simulate_batch.argtypes = [i64, P, P, P, i32, i32, i32, u64, u64, i64, u64, i32,
                                        P, P, P, P, P, P, P, P, P]
        L.or_simulate_batch.restype = ctypes.c_int
        L.or_tel.argtypes = [i64, P, P]
        L.or_tel.restype = i64
        L.or_opt_bruteforce.argtypes = [i64, P, i32, i64, P, P]
        L.or_opt_bruteforce.restype = i64
        L.or_lb_sorted.argtypes = [i64, P, i32]
        L.or_lb_sorted.restype = i64
        L.or_wallclock.argtypes = [i64, P, P, P, i64, i64, i64, i32, i32, P, P, P, P]
        L.or_wallclock.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _req(req) -> np.ndarray:
    r = np.ascontiguousarray(np.asarray(req, dtype=np.int32).reshape(-1, 4))
    return r


def philox4x32_10(ctr, key) -> list[int]:
    """Philox4x32-10 block (Salmon et al., SC'11)."""
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return [int(x) for x in out]


def _cols(rows, k):
    return np.ascontiguousarray(np.array([r[k] for r in rows], dtype=np.int32).reshape(-1))


def projected_occupancy(tp: int, t: int, S, U) -> int:
    """LHS of Eq. 5 at t'.  S = [(s, p, o~)], U = [(s, o~)]."""
    Ss, Sp, So = (_cols(S, k) for k in range(3)) if S else (np.zeros(1, np.int32),) * 3
    Us, Uo = (_cols(U, k) for k in range(2)) if U else (np.zeros(1, np.int32),) * 2
    return int(lib().or_projected_occupancy(tp, t, len(S), _ptr(Ss), _ptr(Sp), _ptr(So),
                                            len(U), _ptr(Us), _ptr(Uo)))


def is_feasible(t: int, budget: int, S, U) -> bool:
    """Eq. 5 for every t' in [t+1, t_max(U)], exhaustive scan."""
    Ss, Sp, So = (_cols(S, k) for k in range(3)) if S else (np.zeros(1, np.int32),) * 3
    Us, Uo = (_cols(U, k) for k in range(2)) if U else (np.zeros(1, np.int32),) * 2
    return bool(lib().or_is_feasible(t, budget, len(S), _ptr(Ss), _ptr(Sp), _ptr(So),
                                     len(U), _ptr(Us), _ptr(Uo)))


def simulate(req, M: int, policy: int = MCSF, alpha=(0, 1), beta_thresh: int = 0,
             seed: int = 0, round_cap: int = 0, gid: int = 0) -> dict:
    """One instance (req rows {a, s, o, o~}, sorted by a) under one policy."""
    r = _req(req)
    n = r.shape[0]
    comp = np.zeros(max(n, 1), dtype=np.int32)
    start = np.zeros(max(n, 1), dtype=np.int32)
    st = np.zeros(7, dtype=np.int64)
    rc = lib().or_simulate(n, _ptr(r), int(M), int(policy), int(alpha[0]), int(alpha[1]),
                           int(beta_thresh), int(seed) & (2**64 - 1), int(round_cap),
                           int(gid) & (2**64 - 1), _ptr(comp), _ptr(start), _ptr(st))
    if rc != 0:
        raise ValueError("oracle: bad policy (unknown id, or alpha-beta with beta_thresh 0 / > 2^32)")
    return dict(completion=comp[:n].copy(), start=start[:n].copy(), tel=int(st[0]),
                rounds=int(st[1]), decision_rounds=int(st[2]), makespan=int(st[3]),
                peak=int(st[4]), evictions=int(st[5]), status=int(st[6]))


def simulate_batch(offset, req, mem, policy: int = MCSF, alpha=(0, 1), beta_thresh: int = 0,
                   seed: int = 0, round_cap: int = 0, gid0: int = 0,
                   nthreads: int | None = None) -> dict:
    """Every instance of a CSR batch, independently, on a pthread pool."""
    off = np.ascontiguousarray(np.asarray(offset, dtype=np.int64))
    r = _req(req)
    m = np.ascontiguousarray(np.asarray(mem, dtype=np.int32))
    ni = m.shape[0]
    nr = int(off[-1])
    nthreads = nthreads or os.cpu_count() or 1
    out = dict(completion=np.zeros(max(nr, 1), np.int32), start=np.zeros(max(nr, 1), np.int32),
               tel=np.zeros(max(ni, 1), np.int64), rounds=np.zeros(max(ni, 1), np.int64),
               decision_rounds=np.zeros(max(ni, 1), np.int64),
               makespan=np.zeros(max(ni, 1), np.int32), peak=np.zeros(max(ni, 1), np.int32),
               evictions=np.zeros(max(ni, 1), np.int64), status=np.zeros(max(ni, 1), np.int32))
    rc = lib().or_simulate_batch(ni, _ptr(off), _ptr(r), _ptr(m), int(policy), int(alpha[0]),
                            int(alpha[1]), int(beta_thresh), int(seed) & (2**64 - 1),
                            int(round_cap), int(gid0) & (2**64 - 1), int(nthreads),
                            _ptr(out["completion"]), _ptr(out["start"]), _ptr(out["tel"]),
                            _ptr(out["rounds"]), _ptr(out["decision_rounds"]),
                            _ptr(out["makespan"]), _ptr(out["peak"]), _ptr(out["evictions"]),
                            _ptr(out["status"]))
    if rc != 0:
        raise ValueError("oracle: bad policy (unknown id, or alpha-beta with beta_thresh 0 / > 2^32)")
    for k in ("completion", "start"):
        out[k] = out[k][:nr]
    for k in ("tel", "rounds", "decision_rounds", "makespan", "peak", "evictions", "status"):
        out[k] = out[k][:ni]
    out["nthreads"] = nthreads
    return out


def tel(req, completion) -> int:
    """TEL = sum_i (c_i - a_i); -1 if any c_i < 0."""
    r = _req(req)
    c = np.ascontiguousarray(np.asarray(completion, dtype=np.int32))
    return int(lib().or_tel(r.shape[0], _ptr(r), _ptr(c)))


def opt_bruteforce(req, M: int, ub: int | None = None):
    """Hindsight optimum of Eqs. 1-4 by exhaustive branch-and-bound.

    Returns (OPT, start vector or None, nodes).  ``ub`` defaults to MC-SF's TEL."""
    r = _req(req)
    n = r.shape[0]
    if ub is None:
        ub = simulate(r, M, MCSF)["tel"]
    start = np.full(max(n, 1), -1, dtype=np.int32)
    nodes = np.zeros(1, dtype=np.int64)
    v = int(lib().or_opt_bruteforce(n, _ptr(r), int(M), int(ub), _ptr(start), _ptr(nodes)))
    if v < 0:
        raise ValueError("oracle.opt_bruteforce: bad instance")
    return v, (start[:n].copy() if v < ub else None), int(nodes[0])


def lb_sorted(req, M: int) -> int:
    """Volume lower bound on OPT for all-at-0 instances (P:212, P:319 argument)."""
    r = _req(req)
    return int(lib().or_lb_sorted(r.shape[0], _ptr(r), int(M)))


def wallclock(req, start, completion, c0: int, c1: int, bin_width: int = 0, n_bins: int = 0,
              trace_len: int = 0) -> dict:
    """NEXT-4: wall clock of a schedule under the affine batch time c0 + c1 tokens (DESIGN Q28)."""
    r = _req(req)
    st = np.ascontiguousarray(np.asarray(start, dtype=np.int32))
    cp = np.ascontiguousarray(np.asarray(completion, dtype=np.int32))
    bins = np.zeros(max(n_bins, 1), np.int64)
    mem = np.zeros(max(trace_len, 1), np.int32)
    tw, mw = np.zeros(1, np.int64), np.zeros(1, np.int64)
    rc = lib().or_wallclock(r.shape[0], _ptr(r), _ptr(st), _ptr(cp), int(c0), int(c1), int(bin_width),
                            int(n_bins), int(trace_len), _ptr(tw), _ptr(mw), _ptr(bins), _ptr(mem))
    return dict(ok=rc == 0, tel_wall=int(tw[0]), makespan_wall=int(mw[0]), bins=bins[:n_bins],
                mem=mem[:trace_len])
