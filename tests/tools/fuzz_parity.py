# Long randomized parity sweep (GPU box): many seeded batches of mixed shapes through every
# policy, flag and size hint of the C ABI, each compared element by element with the oracle.
# Not part of the pytest suite (it runs for minutes); the log goes to gpurun_out/fuzz_parity.log.
#   python tests/tools/fuzz_parity.py [minutes]
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle as O                                   # test infrastructure (allowed here)
import workloads as W
import paper_2502_07115_b200 as K

FIELDS = [("completion", "completion"), ("start", "start"), ("tel", "tel"), ("rounds", "rounds"),
          ("decision_rounds", "decision_rounds"), ("evictions", "evictions"),
          ("makespan", "makespan"), ("peak", "peak_mem"), ("status", "status")]
KIND = {0: "mcsf", 1: "mcbench", 2: "alpha", 3: "alpha_beta", 4: "mcsf_protected"}


def batch(g, i):
    shape = i % 6
    seed = int(g.integers(1, 1 << 30))
    if shape == 0:
        return W.random_small(int(g.integers(100, 3000)), seed, n_max=int(g.integers(1, 130)),
                              M_lo=4, M_hi=64, a_max=int(g.integers(0, 200)),
                              pred_slack=int(g.integers(0, 2)) * 8), "small"
    if shape == 1:
        return W.random_small(int(g.integers(100, 1500)), seed, n_max=int(g.integers(1, 90)),
                              M_lo=20, M_hi=int(g.integers(65, 3000)), a_max=int(g.integers(0, 400)),
                              pred_slack=int(g.integers(0, 2)) * 40), "ring"
    if shape == 2:
        return W.lane_mix(int(g.integers(100, 5000)), seed, n_max=int(g.integers(1, 200)),
                          gap_max=int(g.integers(0, 60)), len_max=int(g.integers(4, 64))), "lane"
    if shape == 3:
        return W.am2(int(g.integers(1000, 20000)), seed), "am2"
    if shape == 4:
        return W.am1(int(g.integers(10, 300)), seed, n=int(g.integers(1, 2000)),
                     M=int(g.integers(8, 65))), "am1"
    return W.c4(int(g.integers(4, 40)), seed), "c4"


def main():
    minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    # --stream: only the streamed host path (P16 rows, MC policies, M <= 64 shapes)
    stream_only = "--stream" in sys.argv
    ctx = K.Context(0)
    g = np.random.default_rng(20251017)
    t_end = time.time() + 60 * minutes
    runs = fails = 0
    i = 0
    with open("gpurun_out/fuzz_parity" + ("_stream" if stream_only else "") + ".log", "w") as log:
        while time.time() < t_end:
            b, shape = batch(g, i if not stream_only else (2, 3, 0)[i % 3])
            i += 1
            pol = int(g.integers(0, 5)) if not stream_only else int(g.integers(0, 2))
            if pol == 4:
                b = W.with_prediction_noise(b, float(g.choice([0.1, 0.2, 0.5])), seed=i)
            alpha = (int(g.integers(0, 4)), 10) if pol >= 2 else (0, 1)
            beta = W.beta_threshold(float(g.choice([0.1, 0.3, 0.6]))) if pol == 3 else 0
            seed = int(g.integers(0, 1 << 40))
            flags = int(g.integers(0, 4))
            measured = bool(g.integers(0, 2))
            hints = (0, 0, 0) if measured else K.hints_of(b)
            o = O.simulate_batch(b.offset, b.req, b.mem, pol, alpha=alpha, beta_thresh=beta, seed=seed)
            p = K.Policy(KIND[pol], alpha, beta, seed, 0, flags)
            # the request-row format and entry point: int32 rows on the device, a packed
            # format when the batch encodes (decoded on the device, + latency16), or the
            # host-buffer entry point (pipelined copies and kernels)
            mode = str(g.choice(["i32", "u16", "u8", "p16", "host", "hostp16"])) if not stream_only else "hostp16"
            if mode in ("u16", "u8", "p16", "hostp16"):
                pk = {"u8": b.packed_u8, "p16": b.packed_p16, "u16": b.packed_u16, "hostp16": b.packed_p16}[mode]()
                if pk is None:
                    mode = "i32"
            if mode == "hostp16":
                # the host entry point with P16 rows: the streamed pipeline for MC policies
                # (M <= 64), flag chunk count drawn too; the chunked pipeline otherwise
                import os
                os.environ["KVSCHED_HOST_STREAM_CHUNKS"] = str(int(g.choice([1, 3, 16, 64])))
                r = {"completion": np.empty(b.n_req, np.int32), "start": np.empty(b.n_req, np.int32),
                     "latency16": np.empty(b.n_req, np.uint16)}
                for k in ("tel", "rounds", "decision_rounds", "evictions"):
                    r[k] = np.empty(b.n_inst, np.int64)
                for k in ("makespan", "peak_mem", "status"):
                    r[k] = np.empty(b.n_inst, np.int32)
                ctx.run_host(b.offset, pk, b.mem, p, r, hints=K.hints_of(b), req_format=K.kvsched.REQ_P16)
                mode = "hp16" + ("s" if "streamed" in ctx.last_kernel() else "c")
            elif mode == "host":
                r = {"completion": np.empty(b.n_req, np.int32), "start": np.empty(b.n_req, np.int32)}
                for k in ("tel", "rounds", "decision_rounds", "evictions"):
                    r[k] = np.empty(b.n_inst, np.int64)
                for k in ("makespan", "peak_mem", "status"):
                    r[k] = np.empty(b.n_inst, np.int32)
                ctx.run_host(b.offset, b.req, b.mem, p, r, hints=K.hints_of(b))
            elif mode == "i32":
                r = K.simulate(ctx, b, p, hints=hints)
            else:
                r = K.simulate(ctx, b, p, hints=hints, packed=mode, latency16=True)
            bad = []
            if "latency16" in r:
                ok_ = np.asarray(o["status"])[np.repeat(np.arange(b.n_inst), np.diff(b.offset))] == 0
                lat = np.minimum(np.asarray(o["completion"]).astype(np.int64) - b.req[:, 0], 65535)[ok_]
                if not np.array_equal(np.asarray(r["latency16"]).astype(np.int64)[ok_], lat):
                    bad.append("latency16")
            for ok, gk in FIELDS:
                x, y = np.asarray(o[ok]).astype(np.int64), np.asarray(r[gk]).astype(np.int64)
                if not np.array_equal(x, y):
                    bad.append(f"{ok}:{int((x != y).sum())}")
            runs += 1
            fails += bool(bad)
            print(f"{i:4d} {shape:5s} {mode:4s} pol={KIND[pol]:14s} alpha={alpha} flags={flags} measured_hints={measured} "
                  f"n_inst={b.n_inst} n_req={b.n_req} -> {'OK' if not bad else 'MISMATCH ' + ' '.join(bad)}",
                  file=log, flush=True)
        print(f"runs {runs} mismatching {fails}", file=log)
    print(f"runs {runs} mismatching {fails}")
    ctx.close()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
