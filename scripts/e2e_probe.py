"""Sensitivity of the host-path (end-to-end) time to what is copied: C5, 10^6 instances."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

b = W.am2(1_000_000, 5)
side = torch.cuda.Stream()
ctx = K.Context(0, stream=side.cuda_stream if "--stream" in sys.argv else None)
pol = K.Policy("mcsf")
hints = K.hints_of(b)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
rows = {"p16": (pin(b.packed_p16()), kv.REQ_P16), "u8": (pin(b.packed_u8()), kv.REQ_U8X4_DELTA),
        "i32": (pin(b.req), kv.REQ_I32X4)}
off, mem = pin(b.offset), pin(b.mem)
def outs(names):
    o = {}
    for k in names:
        n = b.n_req if k in ("completion", "latency16") else b.n_inst
        dt = np.int64 if k in ("tel", "rounds", "decision_rounds", "evictions") else np.uint16 if k == "latency16" else np.int32
        o[k] = pin(np.empty(n, dt))
    return o
full = ["tel", "rounds", "decision_rounds", "evictions", "makespan", "peak_mem", "status", "latency16"]
for fmt in ("p16",):
    for names in (full, ["tel", "status", "latency16"], ["tel", "status"]):
        r, f = rows[fmt]
        o = outs(names)
        ctx.run_host(off, r, mem, pol, o, hints=hints, req_format=f)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            ctx.run_host(off, r, mem, pol, o, hints=hints, req_format=f)
        torch.cuda.synchronize()
        print(fmt, ",".join(names), round((time.perf_counter() - t0) / 5 * 1e3, 3), "ms")
