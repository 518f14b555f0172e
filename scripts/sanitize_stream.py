"""compute-sanitizer target for the streamed host path (round 2): P16 rows decoded by
k_mc_lane<..., p16> and k_mc_small, latency16 written by the kernels, the ordered size-scope
selection, stream memory operations; both MC policies, several chunk counts."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import workloads as W
import paper_2502_07115_b200 as K
import paper_2502_07115_b200.kvsched as kv

ctx = K.Context(0)
b = W.from_instances([W.am2(600, 11).instance(k) for k in range(600)] +
                     [W.lane_mix(60, 12, n_max=130, s_max=8, gap_max=30).instance(k) for k in range(60)])
pk = b.packed_p16()
for chunks in ("1", "7"):
    os.environ["KVSCHED_HOST_STREAM_CHUNKS"] = chunks
    for kind in ("mcsf", "mcbench"):
        outs = {"latency16": np.empty(b.n_req, np.uint16), "tel": np.empty(b.n_inst, np.int64),
                "status": np.empty(b.n_inst, np.int32), "completion": np.empty(b.n_req, np.int32)}
        ctx.run_host(b.offset, pk, b.mem, K.Policy(kind), outs, hints=K.hints_of(b), req_format=kv.REQ_P16)
        print("stream", chunks, kind, ctx.last_kernel(), np.bincount(outs["status"], minlength=4), int(outs["tel"].sum()))
