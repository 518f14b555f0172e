#!/usr/bin/env python
"""bench.py -- MC-SF scheduling rounds/sec over batched instances on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kvsched|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A step is one pass of the whole hot path over one batch: sched_run_instances (MC-SF,
Algorithm 1 of arXiv 2502.07115) over every instance of this rank's shard, plus (N > 1) the
NCCL all_gather of per-instance (TEL, rounds, status) and the all_reduce of totals that the
north star names.  Workload (default) = BASELINE config 5: the Arrival-Model-2 sweep
lambda x M x seed (10^6 instances per GPU; weak scaling: every rank runs its own 10^6).
Inputs are device-resident before timing and larger than L2 (800 MB vs 126 MB).

The JSON line carries the device-timed value, the end-to-end value through the C ABI with
host buffers, the HBM roofline of the simulation kernel, the CPU oracle baseline, clocks
and the kernel launch count.  --impl reference times the oracle (the CPU reference) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads as W  # noqa: E402

METRIC = "MC-SF scheduling rounds/sec over batched instances"
UNIT = "rounds/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kvsched", choices=["kvsched", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c2", "c4", "c3"])
    ap.add_argument("--instances", type=int, default=0,
                    help="instances (0 = config size): of the whole job with --split strong, per GPU with weak")
    ap.add_argument("--split", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's batch (C5: 10^6 instances) is cut across the "
                         "ranks by dist.shard_bounds, balanced by request count; weak: every rank "
                         "runs its own full-size batch")
    ap.add_argument("--dump-results", default="",
                    help="rank 0 saves the gathered per-instance (TEL, rounds, status) rows of the "
                         "last step here (.npy; tests compare 1-rank and N-rank runs)")
    ap.add_argument("--policy", default="mcsf", choices=["mcsf", "mcbench", "alpha", "alpha_beta", "mcsf_protected",
                                                          "mcsf_protected_raise"])
    ap.add_argument("--eps", type=float, default=0.2, help="prediction noise for mcsf_protected (P:519)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-also", action="store_true",
                    help="skip the secondary configs[1] (C2) measurement carried in the line")
    ap.add_argument("--ab", action="store_true",
                    help="also time SCHED_FLAG_PER_ROUND (one Eq. 5 evaluation per round)")
    return ap.parse_args()


def make_workload(name: str, n: int, rank: int, world: int = 1, split: str = "weak"):
    """The config's synthetic batch for this rank and the instance id of its first instance.

    split == "strong": every rank draws the same global batch (rank 0's seed) and keeps the
    contiguous shard [lo, hi) of dist.shard_bounds weighted by request count; its instance
    ids are lo..hi-1, so the alpha-beta RNG and every output equal the 1-GPU run's.
    split == "weak": rank r draws its own full-size batch (ids r*n ...)."""
    if split == "strong" and world > 1:
        from paper_2502_07115_b200 import dist as D
        full, cfg = make_workload(name, n, 0)
        full = full[0]
        bounds = [D.shard_bounds(full.n_inst, world, r, weights=full.sizes()) for r in range(world)]
        lo, hi = bounds[rank]
        cfg.pop("instances_per_gpu", None)
        cfg.update(instances_total_config=full.n_inst, shard=[lo, hi], split="strong",
                   shard_sizes=[b - a for a, b in bounds])
        return (full.slice(lo, hi), lo), cfg
    b, cfg = _make_workload(name, n, rank)
    cfg.update(split=split if world > 1 else "single", shard_sizes=[b.n_inst] * world)
    return (b, rank * b.n_inst), cfg


def _make_workload(name: str, n: int, rank: int):
    if name == "c5":
        n = n or 1_000_000
        return W.am2(n, seed=5, id0=rank * n), dict(workload="C5 AM2 sweep lambda{0.5..1.5} x M{30..50}",
                                                    instances_per_gpu=n, requests_per_instance="Poisson(lambda T), T~U{40..60}")
    if name == "c2":
        n = n or 10_000
        return W.am1(n, seed=2 + 1000 * rank), dict(workload="C2 AM1 n=1000 at t=0, M=40",
                                                    instances_per_gpu=n, requests_per_instance=1000)
    if name == "c4":
        n = n or 20_000
        return W.c4(n, seed=4 + 1000 * rank), dict(workload="C4 trace-shaped n=1000 lambda=2/round M=16492",
                                                   instances_per_gpu=n, requests_per_instance=1000)
    n = n or 4096
    return W.c3(n, seed=3 + 1000 * rank), dict(workload="C3 trace-shaped n=10^4 lambda=2/round M=16492",
                                               instances_per_gpu=n, requests_per_instance=10_000)


def policy_of(K, name):
    if name == "alpha":
        return K.Policy("alpha", (1, 4))
    if name == "alpha_beta":
        return K.Policy("alpha_beta", (1, 5), W.beta_threshold(0.1), seed=1)
    if name in ("mcsf_protected", "mcsf_protected_raise"):
        return K.Policy(name, (1, 10))
    return K.Policy(name)


def oracle_policy(name):
    import oracle
    return {"mcsf": (oracle.MCSF, {}), "mcbench": (oracle.MCBENCH, {}),
            "alpha": (oracle.ALPHA, dict(alpha=(1, 4))),
            "alpha_beta": (oracle.ALPHA_BETA, dict(alpha=(1, 5), beta_thresh=W.beta_threshold(0.1), seed=1)),
            "mcsf_protected": (oracle.MCSF_PROT, dict(alpha=(1, 10))),
            "mcsf_protected_raise": (oracle.MCSF_PROT_RAISE, dict(alpha=(1, 10)))}[name]


def cpu_oracle_rate(batch, policy: str, seconds: float, gid0: int = 0, nthreads: int = 0):
    """The oracle as it stands, on all host cores (or `nthreads`), over a bounded prefix of
    the workload (chunks of 2000 instances sliced without copies; only the oracle call is
    timed)."""
    import oracle
    pol, kw = oracle_policy(policy)
    nthreads = nthreads or os.cpu_count() or 1
    chunk = max(1, min(batch.n_inst, 2000))
    rounds = 0
    insts = 0
    busy = 0.0
    k = 0
    while busy < seconds and k < batch.n_inst:
        sub = batch.slice(k, min(k + chunk, batch.n_inst))
        t0 = time.perf_counter()
        out = oracle.simulate_batch(sub.offset, sub.req, sub.mem, pol, gid0=gid0 + k, nthreads=nthreads, **kw)
        busy += time.perf_counter() - t0
        rounds += int(out["rounds"][out["status"] == 0].sum())
        insts += sub.n_inst
        k += chunk
    return dict(value=rounds / busy, unit=UNIT, cores=nthreads, kind="oracle",
                sample=f"first {insts} instances of the same workload ({rounds} rounds, {busy:.1f} s)",
                instances_per_s=insts / busy)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path(f"/tmp/kvsched_clocks_{os.getpid()}.csv")

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        self.path.unlink(missing_ok=True)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def algorithmic_bytes(batch, fields) -> int:
    """HBM bytes the method must move per launch: request tuples, offsets and budgets in;
    the requested outputs out (DESIGN "Roofline")."""
    b = batch.n_req * 16 + (batch.n_inst + 1) * 8 + batch.n_inst * 4
    for k in fields:
        if k in ("completion", "start"):
            b += batch.n_req * 4
        elif k in ("tel", "rounds", "decision_rounds", "evictions"):
            b += batch.n_inst * 8
        else:
            b += batch.n_inst * 4
    return b


def ncu_record(kernel_name: str) -> dict:
    """The committed ncu --set full capture of this kernel (profiles/ncu_summary.json)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return {}
    try:
        return json.loads(p.read_text()).get("kernels", {}).get(kernel_name, {})
    except Exception:
        return {}


def issue_roofline(rec: dict, sm_mhz: float | None):
    """Instruction issue (one warp instruction per SM sub-partition per clock: 148 SMs x 4
    x f_SM), reported beside the ALU-pipe roofline.  Achieved = warp instructions /
    duration of the committed ncu capture."""
    try:
        inst = float(str(rec["warp_inst"]).replace(",", ""))
        dur = float(rec["duration_ms"]) / 1e3
    except Exception:
        return None
    f = (sm_mhz or 1965.0) * 1e6
    peak = 148 * 4 * f
    return {"bound": "issue", "achieved": inst / dur, "peak": peak, "unit": "warp-inst/s",
            "frac": inst / dur / peak, "source": rec.get("source"), "sm_mhz": sm_mhz or 1965.0}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    (batch, _), cfg = make_workload(args.workload, args.instances, 0)
    if args.policy.startswith("mcsf_protected"):
        batch = W.with_prediction_noise(batch, args.eps, seed=7)
        cfg["prediction_noise_eps"] = args.eps
    per_step = max(args.cpu_seconds / max(args.steps + args.warmup, 1), 0.5)
    for _ in range(args.warmup):
        cpu_oracle_rate(batch, args.policy, per_step)
    vals = [cpu_oracle_rate(batch, args.policy, per_step) for _ in range(args.steps)]
    v = statistics.median([x["value"] for x in vals])
    cfg.update(policy=args.policy, l2="n/a (CPU)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "oracle",
                             "sample": vals[0]["sample"] + " per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2502_07115_b200 as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # KVSCHED_BENCH_BACKEND=gloo + KVSCHED_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo --
    # only to exercise the multi-rank code path on a one-GPU box (never a measurement)
    if os.environ.get("KVSCHED_BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("KVSCHED_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    (batch, id0), cfg = make_workload(args.workload, args.instances, rank, world, args.split)
    if args.policy.startswith("mcsf_protected"):
        batch = W.with_prediction_noise(batch, args.eps, seed=7 + rank)
        cfg["prediction_noise_eps"] = args.eps
    hints = K.hints_of(batch)
    off, req, mem = K.to_device(batch, dev)
    fields = K.kvsched.OUT_FIELDS
    out = K.alloc_outputs(batch.n_inst, batch.n_req, dev, fields)
    stream = torch.cuda.current_stream(dev)
    ctx = K.Context(local, stream=stream.cuda_stream)
    pol = policy_of(K, args.policy)
    shard_sizes = cfg.pop("shard_sizes")
    if world > 1:
        from paper_2502_07115_b200 import dist as D
        res_dtype = D.result_dtype(batch, args.policy)
        # the gather pads every shard to the largest one (strong split: shards differ by a few)
        n_pad = max(shard_sizes)
        gathered = [None, None]

    # N > 1: the north star's only collective -- every rank gathers the per-instance
    # (TEL, rounds, status) of all shards and all ranks reduce the totals (NCCL over NVLink /
    # NVSwitch).  Each step packs its results on the compute stream into one of two
    # buffers and runs the collectives on a side stream, so step k's exchange overlaps step
    # k+1's kernels; a buffer is repacked only after its previous exchange has finished, and
    # the timed region ends after the last exchange.
    if world > 1:
        coll = torch.cuda.Stream(dev)
        packed = [None, None]
        done_ev = [None, None]
        nstep = [0]

    def step():
        ctx.run(off, req, mem, pol, out, id0=id0, hints=hints)
        if world > 1:
            j = nstep[0] % 2
            nstep[0] += 1
            if done_ev[j] is not None:
                stream.wait_event(done_ev[j])
            packed[j] = D.pack_results(out, batch.n_inst, n_pad, dev, res_dtype)
            ready = torch.cuda.Event()
            ready.record(stream)
            packed[j].record_stream(coll)               # allocator: in use on the side stream
            with torch.cuda.stream(coll):
                coll.wait_event(ready)
                gathered[j] = D.gather_results(packed[j])
                D.reduce_totals({k: packed[j][i] for i, k in enumerate(D.RESULT_ROWS)}, batch.n_inst)
                done_ev[j] = torch.cuda.Event()
                done_ev[j].record(coll)

    def join_collectives():
        if world > 1:
            for ev in done_ev:
                if ev is not None:
                    stream.wait_event(ev)

    for _ in range(max(args.warmup, 0)):
        step()
    join_collectives()
    torch.cuda.synchronize(dev)
    rounds_rank = int(out["rounds"][:batch.n_inst].clamp(min=0).sum().item())
    ok_rank = int((out["status"][:batch.n_inst] == 0).sum().item())
    drounds_rank = int(out["decision_rounds"][:batch.n_inst].sum().item())

    clocks = Clocks(local)
    ctx.reset_stats()
    ctx.set_timing(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    join_collectives()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ctx.set_timing(False)
    st = ctx.stats()
    ms = e0.elapsed_time(e1)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([rounds_rank, ok_rank, batch.n_inst], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
    ms_max = float(t_max.item())
    rounds_all, ok_all, inst_all = (int(x) for x in tot.tolist())
    value = rounds_all * args.steps / (ms_max / 1000.0)

    # roofline of the dominant simulation kernel (most device time inside the timed region;
    # CUDA events on the launching stream, per kernel name, from the library's accounting)
    kst = ctx.kernel_stats()
    kname = max(kst, key=lambda k: kst[k][0]) if kst else ctx.last_kernel()
    k_tot_ms, k_launches = kst.get(kname, (st["sim_kernel_ms"], st["sim_kernel_launches"]))
    k_ms = k_tot_ms / max(k_launches, 1)                    # mean duration of one launch
    alg = algorithmic_bytes(batch, fields)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak_gbs = peaks.get("hbm_gbs", 6650.0)
    rec = ncu_record(kname)
    same_launch = rec.get("source", "").find("bench") >= 0 and args.workload == "c5" and args.policy == "mcsf" \
        and batch.n_inst == 1_000_000
    traffic = rec.get("dram_bytes_per_launch") if same_launch else None
    hbm = {"bound": "hbm", "achieved": alg / (k_ms / 1e3) / 1e9, "peak": peak_gbs, "unit": "GB/s",
           "frac": alg / (k_ms / 1e3) / 1e9 / peak_gbs, "alg_bytes_per_launch": alg,
           "peak_source": "measured" if peaks else "fallback"}
    # The simulators are bound by the integer ALU pipe (SWAR / DPX / logic ops), not by HBM:
    # peak = 148 SMs x 4 sub-partitions x 0.5 ALU-pipe warp instructions per clock (the
    # guide's rt_SMSP = 2 for IADD3/LOP3/SHF/PRMT/VIMNMX) at the SM clock measured under load;
    # achieved = the launch's ALU-pipe warp instructions (ncu capture of this same launch
    # configuration: the work is deterministic) / the live mean launch duration.
    f_mhz = (ck or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    alu_peak = 148 * 4 * 0.5 * f_mhz * 1e6
    alu_inst = rec.get("alu_inst")
    if alu_inst is not None and same_launch:
        alu_ach = float(str(alu_inst).replace(",", "")) / (k_ms / 1e3)
        roof = {"bound": "alu", "kernel": kname, "achieved": alu_ach, "peak": alu_peak,
                "unit": "ALU-pipe warp-inst/s", "frac": alu_ach / alu_peak, "traffic": traffic,
                "peak_source": f"derived: 148 x 4 x 0.5/clk x {f_mhz:.0f} MHz (measured SM clock under load)",
                "alu_inst_per_launch": float(str(alu_inst).replace(",", "")),
                "alu_inst_source": rec.get("source")}
    else:
        roof = dict(hbm, kernel=kname, traffic=traffic)
    roof.update(kernel_ms=k_ms, launches_per_step=k_launches / max(args.steps, 1),
                kernel_share_of_step=(k_tot_ms / args.steps) / (ms_max / args.steps) if args.steps else None,
                kernels={k: {"ms_per_step": v[0] / max(args.steps, 1), "launches_per_step": v[1] / max(args.steps, 1)}
                         for k, v in kst.items()},
                kernels_note="CUDA events bracket each launch on its own stream: the side-stream fallbacks "
                             "(k_mc_flatq / k_mc_small beside k_mc_lane, usually an empty or ~1 % list) include "
                             "the wait for SMs held by the main kernel; per-launch work is in the ncu launch list",
                hbm=hbm, issue=issue_roofline(rec, f_mhz) if same_launch else None)

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and world >= 1:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        # Rows on the wire in the narrowest encoding they fit (SCHED_REQ_P16: 2 bytes per
        # request on C5, else uint8 / uint16 deltas, else int32); the schedule comes back as
        # the compact latency16 (c_i - a_i, uint16 per request) plus the per-instance
        # outputs.  start = completion - o and completion = a + latency16 are not copied.
        pk16 = batch.packed_p16()
        pk8 = batch.packed_u8() if pk16 is None else None
        pk = pk8 if pk8 is not None else batch.packed_u16()
        if pk16 is not None:
            fmt, rows, fmt_name = K.kvsched.REQ_P16, pk16.view(np.int16), "p16"
        elif pk8 is not None:
            fmt, rows, fmt_name = K.kvsched.REQ_U8X4_DELTA, pk8.view(np.int8), "u8x4-delta"
        elif pk is not None:
            fmt, rows, fmt_name = K.kvsched.REQ_U16X4_DELTA, pk.view(np.int16), "u16x4-delta"
        else:
            fmt, rows, fmt_name = K.kvsched.REQ_I32X4, batch.req, "i32x4"
        e2e_fields = [k for k in fields if k not in ("start", "completion")] + ["latency16"]
        h_off, h_req, h_mem = pin(batch.offset), pin(rows), pin(batch.mem)
        h_out = {}
        # per-instance outputs field-major in one pinned block per dtype (the int64 four, the
        # int32 three): the library then copies each chunk's fields with one 2-D copy
        i64f = [k for k in e2e_fields if k in K.kvsched.OUT_I64]
        i32f = [k for k in e2e_fields if k not in K.kvsched.OUT_I64 and k not in ("completion", "start", "latency16")]
        for group, dt in ((i64f, torch.int64), (i32f, torch.int32)):
            blk = torch.empty((max(len(group), 1), max(batch.n_inst, 1)), dtype=dt).pin_memory()
            for j, k in enumerate(group):
                h_out[k] = blk[j]
        for k in e2e_fields:
            if k not in h_out:
                n = batch.n_req if k in ("completion", "start", "latency16") else batch.n_inst
                dt = torch.int16 if k == "latency16" else torch.int32
                h_out[k] = torch.empty(max(n, 1), dtype=dt).pin_memory()
        host = {k: v.numpy() for k, v in h_out.items()}
        a_off, a_req, a_mem = h_off.numpy(), h_req.numpy(), h_mem.numpy()
        ctx.run_host(a_off, a_req, a_mem, pol, host, id0=id0, hints=hints, req_format=fmt)      # warm
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            ctx.run_host(a_off, a_req, a_mem, pol, host, id0=id0, hints=hints, req_format=fmt)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        comp_dev = out["completion"][:batch.n_req].cpu().numpy().astype(np.int64)
        lat = host["latency16"][:batch.n_req].view(np.uint16).astype(np.int64)
        same = bool(np.array_equal(host["rounds"][:batch.n_inst], out["rounds"][:batch.n_inst].cpu().numpy())
                    and np.array_equal(batch.req[:, 0].astype(np.int64) + lat, comp_dev))
        if world > 1:                     # every rank's host-path results against its device run
            ok_t = torch.tensor([1 if same else 0], dtype=torch.int64, device=dev)
            dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
            same = bool(ok_t.item())
        h2d = rows.nbytes + (batch.n_inst + 1) * 8 + batch.n_inst * 4
        d2h = sum(v.numel() * v.element_size() for v in h_out.values())
        e2e = {"value": rounds_all * args.e2e_steps / (e_ms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": e_ms / args.e2e_steps, "matches_device_run": bool(same),
               "req_format": fmt_name, "outputs": e2e_fields}

    ab = None
    if args.ab:
        pr = K.Policy(pol.kind, pol.alpha, pol.beta_thresh, pol.seed, pol.round_cap, K.kvsched.FLAG_PER_ROUND)
        ctx.run(off, req, mem, pr, out, id0=id0, hints=hints)
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            ctx.run(off, req, mem, pr, out, id0=id0, hints=hints)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        ab_ms = g0.elapsed_time(g1) / args.steps
        ab = {"per_round_kernel": ctx.last_kernel(), "per_round_ms_per_step": ab_ms,
              "per_round_value": rounds_rank * world / (ab_ms / 1000.0),
              "speedup_of_default": ab_ms / (ms_max / args.steps)}
        # one warp per instance (k_mc_small for every instance) vs the default lane kernel
        pw = K.Policy(pol.kind, pol.alpha, pol.beta_thresh, pol.seed, pol.round_cap,
                      K.kvsched.FLAG_WARP_PER_INSTANCE)
        ctx.run(off, req, mem, pw, out, id0=id0, hints=hints)
        torch.cuda.synchronize(dev)
        g0.record(stream)
        for _ in range(args.steps):
            ctx.run(off, req, mem, pw, out, id0=id0, hints=hints)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        wp_ms = g0.elapsed_time(g1) / args.steps
        ab.update(warp_kernel=ctx.last_kernel(), warp_ms_per_step=wp_ms,
                  warp_value=rounds_rank * world / (wp_ms / 1000.0),
                  speedup_over_warp=wp_ms / (ms_max / args.steps))

    # The other BASELINE configs under the same protocol (inputs resident, CUDA events on the
    # launching stream, max over ranks), reported beside the primary workload: configs[1]
    # (C2: AM1, 10^4 instances of 1000 requests at t=0, M=40), configs[3] (C4: trace-shaped,
    # 2*10^4 instances of 1000 requests, M=16492) and configs[2] (C3: trace-shaped, 4096
    # instances of 10^4 requests); MC-SF.
    also = None
    if not args.no_also and args.workload == "c5" and args.policy == "mcsf":
        also = {}
        for wl, label in (("c2", "C2"), ("c4", "C4"), ("c3", "C3")):
            (b2, id2), cfg2 = make_workload(wl, 0, rank, world, args.split)
            cfg2.pop("shard_sizes", None)
            o2, r2, m2 = K.to_device(b2, dev)
            out2 = K.alloc_outputs(b2.n_inst, b2.n_req, dev, fields)
            h2 = K.hints_of(b2)
            for _ in range(max(args.warmup, 1)):
                ctx.run(o2, r2, m2, pol, out2, id0=id2, hints=h2)
            torch.cuda.synchronize(dev)
            rounds2 = int(out2["rounds"][:b2.n_inst].clamp(min=0).sum().item())
            ok2 = int((out2["status"][:b2.n_inst] == 0).sum().item())
            if world > 1:
                dist.barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.reset_stats()
            ctx.set_timing(True)
            steps2 = args.steps if wl != "c3" else max(1, min(args.steps, 5))
            h0.record(stream)
            for _ in range(steps2):
                ctx.run(o2, r2, m2, pol, out2, id0=id2, hints=h2)
            h1.record(stream)
            torch.cuda.synchronize(dev)
            t2 = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
            n2 = torch.tensor([rounds2, ok2, b2.n_inst], dtype=torch.int64, device=dev)
            if world > 1:
                dist.all_reduce(t2, op=dist.ReduceOp.MAX)
                dist.all_reduce(n2)
            ms2 = float(t2.item())
            ctx.set_timing(False)
            kst2 = ctx.kernel_stats()
            r_all, ok_all2, ni_all = (int(x) for x in n2.tolist())
            also[label] = {"workload": cfg2["workload"], "instances": ni_all, "instances_ok": ok_all2,
                           "value": r_all * steps2 / (ms2 / 1e3), "unit": UNIT, "steps": steps2,
                           "ms_per_step": ms2 / steps2, "rounds_per_step": r_all,
                           "kernel": max(kst2, key=lambda k: kst2[k][0]) if kst2 else ctx.last_kernel(),
                           "kernels_ms_per_step": {k: v[0] / steps2 for k, v in kst2.items()}}
            del o2, r2, m2, out2, b2
            torch.cuda.empty_cache()

    # rank 0: the gathered per-instance rows of the last timed step, in global instance order
    if args.dump_results and rank == 0:
        if world > 1:
            rows = D.unpad(gathered[(nstep[0] - 1) % 2], shard_sizes).to(torch.int64).cpu().numpy()
        else:
            rows = np.stack([out[k][:batch.n_inst].to(torch.int64).cpu().numpy() for k in ("tel", "rounds", "status")])
        np.save(args.dump_results, rows)

    # the oracle on rank 0's host cores, over a bounded prefix of rank 0's shard (at N > 1
    # the other ranks wait at the final barrier; the timed region is over)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rate(batch, args.policy, args.cpu_seconds, gid0=id0)
        one = cpu_oracle_rate(batch, args.policy, min(3.0, args.cpu_seconds / 4), gid0=id0, nthreads=1)
        cpu["single_core"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}

    if rank == 0:
        cfg.update(policy=args.policy, l2="inputs %.0f MB > 126 MB L2 (no flush needed)" % (batch.req.nbytes / 1e6),
                   parallelism=f"instance-sharded x{world}", instances_total=inst_all,
                   instances_ok=ok_all, rounds_per_step=rounds_all,
                   generator=W.GENERATOR_VERSION)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": args.split,
                "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": cfg, "instances_per_s": inst_all * args.steps / (ms_max / 1000.0),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": ck,
                "gpu_launches": st["launches"], "decision_rounds_per_step": drounds_rank * world,
                "ab": ab, "other_configs": also}
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        dist.barrier()                  # rank 0 may still be timing the oracle
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
