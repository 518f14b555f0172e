#!/usr/bin/env python
"""Run every BASELINE.json config through the GPU path (C ABI), check sampled instances
against the CPU oracle, and report throughput plus the statistic the config is quoted for.

    python tests/tools/configs_report.py [--out profiles/r01/configs_report.json] [--quick]

C1  tiny (n=8, M=16): MC-SF TEL vs the brute-force hindsight optimum (Eqs. 1-4)
C2  AM1 (n=1000 at t=0, M=40): TEL(MC-SF) / LB_sorted, an upper bound on the ratio to OPT
C3  trace-shaped n=10^4, M=16492, lambda in {0.4, 2.0}/round
C4  trace-shaped n=1000: the 8 policies of Table 1, average latency in rounds
C5  AM2 sweep lambda x M x seed, 10^6 instances
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (test infrastructure: parity sampling and OPT only)
import paper_2502_07115_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

POL = {"mcsf": oracle.MCSF, "mcbench": oracle.MCBENCH, "alpha": oracle.ALPHA, "alpha_beta": oracle.ALPHA_BETA,
       "mcsf_protected": oracle.MCSF_PROT, "mcsf_protected_raise": oracle.MCSF_PROT_RAISE}


def oracle_rate(b, kind, seconds=4.0, **kw):
    """The oracle on all host cores over a bounded prefix of the batch (rounds/s)."""
    import os
    chunk, k, busy, rounds, insts = max(1, min(b.n_inst, 500)), 0, 0.0, 0, 0
    while busy < seconds and k < b.n_inst:
        sub_ = b.slice(k, min(k + chunk, b.n_inst))
        t0 = time.perf_counter()
        o = oracle.simulate_batch(sub_.offset, sub_.req, sub_.mem, POL[kind], gid0=k, **kw)
        busy += time.perf_counter() - t0
        rounds += int(o["rounds"][o["status"] == 0].sum())
        insts += sub_.n_inst
        k += chunk
    return {"rounds_per_s": rounds / busy, "cores": os.cpu_count(), "sample_instances": insts}


def gpu(ctx, b, policy, reps=3):
    dev = torch.device("cuda", 0)
    off, req, mem = K.to_device(b, dev)
    out = K.alloc_outputs(b.n_inst, b.n_req, dev)
    hints = K.hints_of(b)
    ctx.run(off, req, mem, policy, out, hints=hints)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.reset_stats()
    ctx.set_timing(True)
    e0.record()
    for _ in range(reps):
        ctx.run(off, req, mem, policy, out, hints=hints)
    e1.record()
    torch.cuda.synchronize()
    ctx.set_timing(False)
    kst = ctx.kernel_stats()
    ms = e0.elapsed_time(e1) / reps
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["completion"] = res["completion"][:b.n_req]
    for k in ("tel", "rounds", "decision_rounds", "evictions", "makespan", "peak_mem", "status"):
        res[k] = res[k][:b.n_inst]
    # the kernel with the most device time (a call may launch several)
    return res, ms, max(kst, key=lambda k: kst[k][0]) if kst else ctx.last_kernel()


def sample_parity(b, g, policy, kind, n_sample, seed=0):
    ks = np.random.default_rng(seed).choice(b.n_inst, min(n_sample, b.n_inst), replace=False)
    bad = 0
    for k in ks:
        req, M = b.instance(int(k))
        o = oracle.simulate(req, M, POL[kind], alpha=policy.alpha, beta_thresh=policy.beta_thresh,
                            seed=policy.seed, gid=int(k))
        lo, hi = int(b.offset[k]), int(b.offset[k + 1])
        ok = (np.array_equal(o["completion"], g["completion"][lo:hi]) and o["tel"] == g["tel"][k]
              and o["rounds"] == g["rounds"][k] and o["status"] == g["status"][k]
              and o["peak"] == g["peak_mem"][k] and o["decision_rounds"] == g["decision_rounds"][k]
              and o["evictions"] == g["evictions"][k])
        bad += not ok
    return {"sampled": len(ks), "mismatches": bad}


def summarize(b, g, ms, kname):
    ok = g["status"] == 0
    rounds = int(g["rounds"][ok].sum())
    return {"instances": b.n_inst, "requests": b.n_req, "kernel": kname, "ms": ms,
            "rounds": rounds, "rounds_per_s": rounds / (ms / 1e3), "instances_per_s": b.n_inst / (ms / 1e3),
            "status_counts": np.bincount(g["status"], minlength=4).tolist()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02" / "configs_report.json"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    q = a.quick
    ctx = K.Context(0)
    report = {}

    # C1: tiny instances vs brute-force OPT
    t0 = time.time()
    b = W.c1(2000 if q else 10_000, 11, "b")
    pol = K.Policy("mcsf")
    g, ms, kn = gpu(ctx, b, pol)
    r = summarize(b, g, ms, kn)
    ratios, n_opt = [], 0
    for k in range(min(b.n_inst, 500 if q else 3000)):
        req, M = b.instance(k)
        opt, _, _ = oracle.opt_bruteforce(req, M, int(g["tel"][k]))
        ratios.append(g["tel"][k] / opt)
        n_opt += g["tel"][k] == opt
    r["tel_over_opt"] = {"n": len(ratios), "mean": float(np.mean(ratios)), "max": float(np.max(ratios)),
                         "exact_optimum": int(n_opt), "never_below_opt": bool(min(ratios) >= 1.0)}
    r["parity"] = sample_parity(b, g, pol, "mcsf", 2000)
    r["oracle"] = oracle_rate(b, "mcsf")
    report["C1"] = r
    print("C1", json.dumps(r), f"({time.time() - t0:.0f}s)", flush=True)

    # C2: AM1 n=1000, M=40: TEL / LB_sorted
    b = W.am1(200 if q else 10_000, 2)
    g, ms, kn = gpu(ctx, b, pol)
    r = summarize(b, g, ms, kn)
    dev = torch.device("cuda", 0)
    off, req, mem = K.to_device(b, dev)
    lbt = torch.empty(b.n_inst, dtype=torch.int64, device=dev)
    ctx.lb_sorted(off, req, mem, lbt, hints=K.hints_of(b))          # NEXT-2, GPU part
    torch.cuda.synchronize()
    lb = lbt.cpu().numpy()
    ub = g["tel"] / lb
    r["tel_over_lb_sorted"] = {"instances": b.n_inst, "mean": float(ub.mean()), "max": float(ub.max()),
                               "min": float(ub.min()), "first_200_seeds_mean": float(ub[:200].mean()),
                               "lb_parity_sampled": int(sum(lb[k] == oracle.lb_sorted(*b.instance(k))
                                                            for k in range(64)))}
    r["parity"] = sample_parity(b, g, pol, "mcsf", 64)
    r["oracle"] = oracle_rate(b, "mcsf")
    report["C2"] = r
    print("C2", json.dumps(r), flush=True)

    # C3: trace-shaped n=10^4, both demand levels
    for lam in (0.4, 2.0):
        b = W.c3(256 if q else 4096, 3, lam)
        for kind in ("mcsf", "mcbench"):
            g, ms, kn = gpu(ctx, b, K.Policy(kind), reps=1)
            r = summarize(b, g, ms, kn)
            ok = g["status"] == 0
            r["avg_latency_rounds"] = float(g["tel"][ok].sum() / (b.n_req / b.n_inst * ok.sum()))
            r["parity"] = sample_parity(b, g, K.Policy(kind), kind, 16)
            r["oracle"] = oracle_rate(b, kind)
            report[f"C3 lambda={lam} {kind}"] = r
            print("C3", lam, kind, json.dumps(r), flush=True)

    # C4: Table 1's eight policies
    b = W.c4(10_000 if q else 100_000, 4)
    for name, kind, alpha, beta in W.C4_POLICIES:
        pol = K.Policy(kind, alpha or (0, 1), W.beta_threshold(beta or 0.0), 2025)
        g, ms, kn = gpu(ctx, b, pol, reps=1)
        r = summarize(b, g, ms, kn)
        ok = g["status"] == 0
        lat = g["tel"][ok] / 1000.0
        r["avg_latency_rounds"] = {"mean": float(lat.mean()), "sd": float(lat.std()), "max": float(lat.max()),
                                   "min": float(lat.min()), "livelock": int((g["status"] == 2).sum())}
        r["evictions_total"] = int(g["evictions"].sum())
        r["parity"] = sample_parity(b, g, pol, kind, 32)
        r["oracle"] = oracle_rate(b, kind, alpha=pol.alpha, beta_thresh=pol.beta_thresh, seed=pol.seed)
        report[f"C4 {name}"] = r
        print("C4", name, json.dumps(r), flush=True)

    # NEXT-1: prediction noise, protected MC-SF (alpha = 0.1) under Q26 and Q26b
    bn = W.c4(2000 if q else 20_000, 4)
    for eps in (0.2, 0.5, 0.8):
        nb = W.with_prediction_noise(bn, eps, seed=7)
        for kind in ("mcsf_protected", "mcsf_protected_raise"):
            pol = K.Policy(kind, (1, 10))
            g, ms, kn = gpu(ctx, nb, pol, reps=1)
            r = summarize(nb, g, ms, kn)
            ok = g["status"] == 0
            r["avg_latency_rounds"] = float((g["tel"][ok] / 1000.0).mean()) if ok.any() else None
            r["completed"] = int(ok.sum())
            r["parity"] = sample_parity(nb, g, pol, kind, 16)
            report[f"C4 noise eps={eps} {kind}"] = r
            print("C4noise", eps, kind, json.dumps(r), flush=True)

    # NEXT-4: wall clock of the C4 MC-SF and MC-Benchmark schedules under an affine batch time
    # (placeholder constants: 20 ms per batch + 0.05 ms per token; only ratios are claimed)
    dev = torch.device("cuda", 0)
    off, req, mem = K.to_device(b, dev)
    wall = {}
    for kind in ("mcsf", "mcbench"):
        out = K.alloc_outputs(b.n_inst, b.n_req, dev)
        ctx.run(off, req, mem, K.Policy(kind), out, hints=K.hints_of(b))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w = ctx.wallclock(off, req, mem, out["start"], out["completion"], 20_000, 50, 1_000_000, 64, 0)
        e1.record()
        torch.cuda.synchronize()
        tw = w["tel_wall"].cpu().numpy()
        wall[kind] = {"avg_latency_s": float(tw.mean() / 1000 / 1e6), "kernel_ms": e0.elapsed_time(e1),
                      "first_instance_tokens_per_s_first_10_bins": w["bins"][0, :10].cpu().tolist()}
        if kind == "mcsf":
            st, cp = out["start"][:1000].cpu().numpy(), out["completion"][:1000].cpu().numpy()
            o = oracle.wallclock(b.req[:1000], st, cp, 20_000, 50, 1_000_000, 64, 0)
            wall[kind]["instance0_matches_oracle"] = o["tel_wall"] == int(tw[0])
    wall["mcsf_over_mcbench_avg_latency"] = wall["mcsf"]["avg_latency_s"] / wall["mcbench"]["avg_latency_s"]
    report["C4 wall clock (NEXT-4)"] = wall
    print("C4wall", json.dumps(wall), flush=True)

    # C5: the sweep (per grid cell mean TEL / n)
    b = W.am2(200_000 if q else 1_000_000, 5)
    pol = K.Policy("mcsf")
    g, ms, kn = gpu(ctx, b, pol)
    r = summarize(b, g, ms, kn)
    r["parity"] = sample_parity(b, g, pol, "mcsf", 500)
    r["oracle"] = oracle_rate(b, "mcsf")
    report["C5"] = r
    print("C5", json.dumps(r), flush=True)

    # NEXT-3: the C5 sweep generated on the device from the counter spec, then simulated
    spec = W.Am2Spec(seed=5)
    n = 200_000 if q else 1_000_000
    off, req, mem, n_req = ctx.gen_am2(n, spec)          # warm-up (allocations)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    off, req, mem, n_req = ctx.gen_am2(n, spec)
    e1.record()
    out = K.alloc_outputs(n, n_req, torch.device("cuda", 0))
    hints = (int(torch.diff(off).max().item()), max(spec.Ms), max(spec.Ms) - spec.s_lo)
    ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=hints)      # warm-up (scratch allocations)
    torch.cuda.synchronize()
    e1b = torch.cuda.Event(enable_timing=True)
    e1b.record()
    ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=hints)
    e2.record()
    torch.cuda.synchronize()
    rounds = int(out["rounds"][:n].clamp(min=0).sum().item())
    hb = W.am2_counter(2000, spec)
    r = {"instances": n, "requests": n_req, "generate_ms": e0.elapsed_time(e1), "simulate_ms": e1b.elapsed_time(e2),
         "generated_instances_per_s": n / (e0.elapsed_time(e1) / 1e3),
         "rounds_per_s_simulation": rounds / (e1b.elapsed_time(e2) / 1e3),
         "bytes_match_host_reference_first_2000": bool(np.array_equal(req[:hb.n_req].cpu().numpy(), hb.req))}
    report["C5 generated on device (NEXT-3)"] = r
    print("C5gen", json.dumps(r), flush=True)

    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(report, indent=1))
    ctx.close()


if __name__ == "__main__":
    main()
