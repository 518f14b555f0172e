"""compute-sanitizer targets added with the lane kernel: k_mc_lane at every profile width
(both policies), its k_mc_small fallback list, the compact u8 rows / latency16 path and the
multi-stream host pipeline."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

ctx = K.Context(0)
for len_max in (12, 28, 48, 63):
    b = W.lane_mix(300, len_max, len_max=len_max, gap_max=6)
    for kind in ("mcsf", "mcbench"):
        g = K.simulate(ctx, b, K.Policy(kind), hints=K.hints_of(b))
        print("lane", len_max, kind, ctx.last_kernel(), np.bincount(g["status"], minlength=4))
mix = W.from_instances([b.instance(k) for k in range(50)] +
                       [W.lane_mix(3, 1, n_max=300).instance(k) for k in range(3)] +
                       [W.lane_mix(5, 2, s_max=12, M_lo=20).instance(k) for k in range(5)] +
                       [([[0, 2, 3, 9], [0, 1, 5, 5]], 20), ([[3, 1, 1, 1], [2, 1, 1, 1]], 10)])
g = K.simulate(ctx, mix, K.Policy("mcsf"), hints=K.hints_of(mix))
print("mix", np.bincount(g["status"], minlength=4))
for kind in ("mcsf", "mcbench"):                       # k_mc_flat (simultaneous arrivals, n > 96)
    f = W.from_instances([W.am1(6, 9, n=300, M=40).instance(k) for k in range(6)] +
                         [W.lane_mix(4, 3, n_max=200, gap_max=2).instance(k) for k in range(4)])
    g = K.simulate(ctx, f, K.Policy(kind), hints=K.hints_of(f))
    print("flat", kind, np.bincount(g["status"], minlength=4))
c = W.am2(400, 3)
g = K.simulate(ctx, c, K.Policy("mcsf"), hints=K.hints_of(c), packed="u8", latency16=True)
print("u8", int(g["latency16"].max()))
os.environ["KVSCHED_HOST_CHUNK_ROWS"] = "2000"
outs = {"latency16": np.empty(c.n_req, np.uint16), "tel": np.empty(c.n_inst, np.int64),
        "status": np.empty(c.n_inst, np.int32)}
ctx.run_host(c.offset, c.packed_u8(), c.mem, kv.Policy("mcsf"), outs, hints=K.hints_of(c),
             req_format=kv.REQ_U8X4_DELTA)
print("done", int(outs["tel"].sum()))
