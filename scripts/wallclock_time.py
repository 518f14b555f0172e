"""Time sched_wallclock on 10^5 C4 MC-SF schedules (experiments: window size)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
import paper_2502_07115_b200 as K

b = W.c4(100_000, 4)
dev = torch.device("cuda", 0)
ctx = K.Context(0)
off, req, mem = K.to_device(b, dev)
out = K.alloc_outputs(b.n_inst, b.n_req, dev)
ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=K.hints_of(b))
args = (off, req, mem, out["start"], out["completion"], 20000, 50)
for _ in range(2):
    r = ctx.wallclock(*args, bin_width=1000000, n_bins=8)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    r = ctx.wallclock(*args, bin_width=1000000, n_bins=8)
e1.record(); torch.cuda.synchronize()
print("wallclock ms", e0.elapsed_time(e1) / 5, int(r["tel_wall"][:b.n_inst].sum().item()))
