"""reproduce the bench's order: device-path runs on a torch stream, then the streamed host path"""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

variant = sys.argv[1]
dev = torch.device("cuda", 0)
b = W.am2(int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000, 5)
hints = K.hints_of(b)
stream = torch.cuda.current_stream(dev)
ctx = K.Context(0, stream=stream.cuda_stream) if "torchstream" in variant else K.Context(0)
if "device" in variant:
    off, req, mem = K.to_device(b, dev)
    out = K.alloc_outputs(b.n_inst, b.n_req, dev, K.kvsched.OUT_FIELDS)
    for _ in range(2):
        ctx.run(off, req, mem, K.Policy("mcsf"), out, hints=hints)
    torch.cuda.synchronize()
    print("device done", flush=True)
pk = b.packed_p16().view(np.int16)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
h_off, h_req, h_mem = pin(b.offset), pin(pk), pin(b.mem)
outs = {"latency16": torch.empty(b.n_req, dtype=torch.int16).pin_memory().numpy()}
for k in ("tel", "rounds", "decision_rounds", "evictions"):
    outs[k] = torch.empty(b.n_inst, dtype=torch.int64).pin_memory().numpy()
for k in ("makespan", "peak_mem", "status"):
    outs[k] = torch.empty(b.n_inst, dtype=torch.int32).pin_memory().numpy()
os.environ["KVSCHED_HOST_STREAM"] = "1"
for i in range(2):
    t = time.time()
    try:
        ctx.run_host(h_off.numpy(), h_req.numpy(), h_mem.numpy(), kv.Policy("mcsf"), outs, hints=hints, req_format=kv.REQ_P16)
        err = "ok"
    except Exception as e:
        err = str(e)[:200]
    print(variant, i, f"{time.time() - t:.3f}s", err, flush=True)
