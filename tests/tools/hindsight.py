#!/usr/bin/env python
"""NEXT-2: MC-SF against the best hindsight schedule found by search, on the
paper's own synthetic experiments: Arrival Model 1 (n~U{40..60} at t=0) and
Arrival Model 2 (Poisson lambda~U[0.5,1.5] over T~U{40..60}), M~U{30..50}, s~U{1..5},
o~U{1..M-s}, 200 trials each.  Test infrastructure (uses the CPU oracle for MC-SF).

TEL(best found) >= OPT, so each reported ratio TEL(MC-SF)/TEL(best) is a LOWER bound on the
paper's TEL(MC-SF)/OPT.  The search is calibrated on C1 (n = 8), where the brute-force OPT
(oracle.opt_bruteforce, pinned against scipy's MILP) is known.

    python tests/tools/hindsight.py [--trials 200] [--iters 40000] [--out profiles/r02/hindsight.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time
from multiprocessing import Pool
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
LIB = HERE / "libhindsight.so"


def build():
    src = HERE / "hindsight.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", str(src), "-o", str(LIB)])


def _lib():
    L = ctypes.CDLL(str(LIB))
    P = ctypes.c_void_p
    L.hs_search.argtypes = [ctypes.c_int, P, ctypes.c_int, P, ctypes.c_int64, ctypes.c_uint64]
    L.hs_search.restype = ctypes.c_int64
    return L


def one(args):
    req, M, iters, seed, want_opt = args
    import oracle
    req = np.ascontiguousarray(req, np.int32)
    mc = oracle.simulate(req, M, oracle.MCSF)
    start = np.ascontiguousarray(mc["start"], np.int32)
    best = int(_lib().hs_search(len(req), req.ctypes.data, int(M), start.ctypes.data, int(iters), int(seed)))
    # the returned schedule must satisfy Eqs. 2-3 (p >= a, memory <= M every round)
    prof = np.zeros(int(start.max(initial=0) + req[:, 2].max(initial=0)) + 2, np.int64)
    for i in range(len(req)):
        p, s, o = int(start[i]), int(req[i, 1]), int(req[i, 2])
        assert p >= req[i, 0]
        prof[p + 1:p + o + 1] += s + np.arange(1, o + 1)
    assert prof.max(initial=0) <= M and int((start + req[:, 2] - req[:, 0]).sum()) == best
    opt = oracle.opt_bruteforce(req, M, mc["tel"])[0] if want_opt else None
    return mc["tel"], best, opt, len(req)


def study(batch, iters, want_opt=False, procs=None):
    jobs = [(batch.instance(k)[0], batch.instance(k)[1], iters, 1000 + k, want_opt) for k in range(batch.n_inst)]
    with Pool(procs or os.cpu_count()) as pool:
        res = pool.map(one, jobs, chunksize=1)
    mc = np.array([r[0] for r in res], float)
    best = np.array([r[1] for r in res], float)
    ratio = mc / best
    out = {"trials": batch.n_inst, "n_mean": float(np.mean([r[3] for r in res])),
           "mcsf_over_best_found": {"mean": float(ratio.mean()), "max": float(ratio.max()), "min": float(ratio.min()),
                                    "mcsf_equals_best_found": int((ratio == 1.0).sum())},
           "iterations_per_trial": iters}
    if want_opt:
        opt = np.array([r[2] for r in res], float)
        out["best_found_equals_opt"] = int((best == opt).sum())
        out["mcsf_over_opt"] = {"mean": float((mc / opt).mean()), "max": float((mc / opt).max()),
                                "mcsf_equals_opt": int((mc == opt).sum())}
    return out, ratio.tolist()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=200)
    ap.add_argument("--iters", type=int, default=40000)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02" / "hindsight.json"))
    a = ap.parse_args()
    build()
    import oracle
    oracle.build()
    import workloads as W
    report = {"paper": {"AM1": {"mean": 1.005, "max": 1.074, "mcsf_equals_opt": 114, "trials": 200, "cite": "PAPER.md:433"},
                        "AM2": {"mean": 1.047, "max": 1.227, "trials": 200, "cite": "PAPER.md:440"}}}
    t0 = time.time()
    report["calibration_C1"], _ = study(W.c1(300, 11, "b"), a.iters // 4, want_opt=True)
    print("C1", report["calibration_C1"], f"{time.time() - t0:.0f}s", flush=True)
    for name, b in (("AM1", W.am1_paper(a.trials, 20)), ("AM2", W.am2_paper(a.trials, 21))):
        t0 = time.time()
        report[name], report[name + "_ratios"] = study(b, a.iters)
        report[name]["seconds"] = time.time() - t0
        print(name, report[name], flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
