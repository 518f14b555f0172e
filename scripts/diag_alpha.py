import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import workloads as W, oracle as O, paper_2502_07115_b200 as K
ctx = K.Context(0)
b = W.c4(2000, 4)
for alpha in ((1, 4), (3, 10), (1, 10)):
    for kind in ("alpha", "alpha_beta"):
        p = K.Policy(kind, alpha, W.beta_threshold(0.1), 1)
        g = K.simulate(ctx, b, p, hints=K.hints_of(b))
        torch.cuda.synchronize()
        t0 = time.time(); g = K.simulate(ctx, b, p, hints=K.hints_of(b)); t1 = time.time()
        print(kind, alpha, f"{t1-t0:.3f}s", np.bincount(g["status"]), "drounds max", g["decision_rounds"].max(),
              "evictions sum", g["evictions"].sum(), "rounds sum", g["rounds"][g["status"] == 0].sum(), flush=True)
        bad = np.argsort(-g["decision_rounds"])[:3]
        for k in bad:
            print("   inst", k, "status", g["status"][k], "drounds", g["decision_rounds"][k], "evict", g["evictions"][k])
