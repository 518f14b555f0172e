"""Small runs of every kernel variant for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2502_07115_b200 as K

ctx = K.Context(0)
batches = [W.am2(300, 1), W.random_small(200, 2, n_max=50, M_lo=4, M_hi=64, a_max=40, pred_slack=5),
           W.am1(2, 3, n=1500, M=40), W.random_small(200, 4, n_max=60, M_lo=10, M_hi=300, a_max=40),
           W.c4(4, 5)]
for b in batches:
    for kind in ("mcsf", "mcbench", "alpha", "alpha_beta"):
        if kind == "mcsf" and b.req[:, 3].max() > 0 and (b.req[:, 3] != b.req[:, 2]).any() and b.max_mem() > 64:
            continue
        for flags in (0, 1):
            p = K.Policy(kind, (1, 10), W.beta_threshold(0.3), 7, 0, flags)
            g = K.simulate(ctx, b, p, hints=K.hints_of(b))
            print(b.name, kind, flags, ctx.last_kernel(), np.bincount(g["status"], minlength=4), flush=True)
off, req, _ = K.to_device(batches[0], torch.device("cuda", 0))
comp = torch.zeros(batches[0].n_req, dtype=torch.int32, device="cuda")
tel = torch.empty(batches[0].n_inst, dtype=torch.int64, device="cuda")
ctx.latency(off, req, comp, tel, None)
torch.cuda.synchronize()
print("done")
