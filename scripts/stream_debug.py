"""streamed host path: time one call at growing sizes; a call far above the chunked path's
time means the per-chunk flags were not set while the lane kernel ran."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

ctx = K.Context(0)
for n in (300_000, 1_000_000):
    b = W.am2(n, 5)
    pk = b.packed_p16()
    rows = pk.view(np.int16)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    h_off, h_req, h_mem = pin(b.offset), pin(rows), pin(b.mem)
    outs = {"latency16": torch.empty(b.n_req, dtype=torch.int16).pin_memory().numpy()}
    for k in ("tel", "rounds", "decision_rounds", "evictions"):
        outs[k] = torch.empty(b.n_inst, dtype=torch.int64).pin_memory().numpy()
    for k in ("makespan", "peak_mem", "status"):
        outs[k] = torch.empty(b.n_inst, dtype=torch.int32).pin_memory().numpy()
    for mode in ("1", "1", "0", "1"):
        os.environ["KVSCHED_HOST_STREAM"] = mode
        t = time.time()
        try:
            ctx.run_host(h_off.numpy(), h_req.numpy(), h_mem.numpy(), kv.Policy("mcsf"), outs,
                         hints=K.hints_of(b), req_format=kv.REQ_P16)
            err = "ok"
        except Exception as e:
            err = str(e)[:200]
        print(n, "stream" if mode == "1" else "chunked", f"{time.time() - t:.3f}s", err,
              int(outs["tel"].sum()), flush=True)
