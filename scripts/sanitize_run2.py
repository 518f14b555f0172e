"""compute-sanitizer targets added after the first pass: k_prot, k_lb_sorted, the generator
kernels, the pipelined host path and the full-ring rerun."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

ctx = K.Context(0)
b = W.with_prediction_noise(W.random_small(150, 2, n_max=40, M_lo=10, M_hi=300, a_max=30), 0.4, seed=1)
g = K.simulate(ctx, b, K.Policy("mcsf_protected", (1, 10)), hints=K.hints_of(b))
print("prot", ctx.last_kernel(), np.bincount(g["status"], minlength=4))
many = W.from_instances([([[0, 1, 2100, 2100]] * 40, 200000), ([[0, 2, 30, 30]], 100)])
for kind in ("mcsf", "alpha_beta", "mcsf_protected"):
    g = K.simulate(ctx, many, K.Policy(kind, (1, 10), 2**30, 3), hints=K.hints_of(many))
    print("rerun", kind, g["status"])
a = W.am1(8, 3)
off, req, mem = K.to_device(a, torch.device("cuda", 0))
lb = torch.empty(a.n_inst, dtype=torch.int64, device="cuda")
ctx.lb_sorted(off, req, mem, lb, hints=K.hints_of(a))
off, req, mem, n = ctx.gen_am2(300, W.Am2Spec(seed=9), id0=5)
torch.cuda.synchronize()
os.environ["KVSCHED_HOST_CHUNK_ROWS"] = "300"
h = W.am2(200, 4)
outs = {"completion": np.empty(h.n_req, np.int32), "tel": np.empty(h.n_inst, np.int64),
        "status": np.empty(h.n_inst, np.int32)}
ctx.run_host(h.offset, h.req, h.mem, kv.Policy("mcsf"), outs, hints=K.hints_of(h))
print("done", int(lb[0].item()), n)
