"""C3 tail diagnosis: the k_mc_ring time of the whole batch vs. the longest instances run
alone (one per SM, four per SM) and the shortest ones; kernel times from the library's
per-kernel CUDA-event stats."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_07115_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

K.load()
ctx = K.Context(0)
ctx.set_timing(True)
b = W.c3(4096, seed=3)
pol = K.Policy("mcsf")


def run(batch, label, reps=2):
    for _ in range(reps):
        ctx.reset_stats()
        g = K.simulate(ctx, batch, pol, hints=K.hints_of(batch))
    ks = ctx.kernel_stats()
    ring = {k: round(v[0], 3) for k, v in ks.items()}
    print(label, batch.n_inst, "rounds mean/max", int(g["rounds"].mean()), int(g["rounds"].max()), ring, flush=True)
    return g


g = run(b, "all")
order = np.argsort(-g["rounds"])
for n_top in (148, 592, 1184, 2368):
    run(b.subset(np.sort(order[:n_top])), f"longest {n_top}")
run(b.subset(np.sort(order[-2368:])), "shortest 2368")
