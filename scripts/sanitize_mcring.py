"""compute-sanitizer targets for the 16-bit MC ring path (k_mc_prep + k_mc_ring, the bulk-copy
arrival staging): C4-shaped batches, ragged budgets, o~ > o (k_prot hand-off), windows past
the ring (long list and the full-ring rerun) and an instance breaking the size hint."""
import sys
sys.path.insert(0, '.')
import numpy as np
import workloads as W
import paper_2502_07115_b200 as K

ctx = K.Context(0)
for kind in ("mcsf", "mcbench"):
    for b in (W.c4(24, 5), W.random_small(200, 7, n_max=90, M_lo=70, M_hi=400, a_max=60),
              W.random_small(100, 8, n_max=40, M_lo=70, M_hi=300, a_max=10, pred_slack=9)):
        g = K.simulate(ctx, b, K.Policy(kind), hints=K.hints_of(b))
        print(kind, b.name, ctx.last_kernel(), np.bincount(g["status"], minlength=4))
    many = W.from_instances([([[0, 1, 2100, 2100]] * 40 + [[5, 3, 50, 50], [9, 2, 2500, 2500]], 200000),
                             ([[0, 3, 700, 700], [1, 2, 3000, 3000], [2, 1, 5, 5]], 4000)])
    g = K.simulate(ctx, many, K.Policy(kind), hints=K.hints_of(many))
    print(kind, "long", np.bincount(g["status"], minlength=4))
    big = W.from_instances([([[0, 1, 5, 5]] * 400, 300)] + [W.random_small(20, 9, n_max=15, M_lo=70,
                                                                            M_hi=200).instance(k) for k in range(20)])
    g = K.simulate(ctx, big, K.Policy(kind), hints=(20, 300, 63))
    print(kind, "hint", np.bincount(g["status"], minlength=4))
print("done")
