"""DESIGN Q26 vs Q26b on C4 with prediction noise, on the CPU oracle:
protected MC-SF (alpha = 0.1) keeping each request's o^ across clearings (Q26) or raising it
to the tokens the request is known to need when it is cleared (Q26b), against MC-Benchmark
(FCFS, true o) and MC-SF with exact predictions.  Reports livelocks and the average
end-to-end latency (TEL/n, rounds) over the completed instances."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import oracle as O
import workloads as W

n_inst = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
base = W.c4(n_inst, 4)
def stats(o, b):
    ok = o["status"] == 0
    lat = o["tel"][ok] / np.diff(b.offset)[ok]
    return dict(ok=int(ok.sum()), livelock=int((o["status"] == 2).sum()),
                mean_latency=float(lat.mean()) if ok.any() else None,
                evictions=float(o["evictions"].mean()))
print("mcsf exact", stats(O.simulate_batch(base.offset, base.req, base.mem, O.MCSF), base))
print("mcbench", stats(O.simulate_batch(base.offset, base.req, base.mem, O.MCBENCH), base))
for eps in (0.2, 0.5, 0.8):
    b = W.with_prediction_noise(base, eps, seed=7)
    for pol, name in ((O.MCSF_PROT, "Q26 keep o^"), (O.MCSF_PROT_RAISE, "Q26b raise o^")):
        t = time.time()
        o = O.simulate_batch(b.offset, b.req, b.mem, pol, alpha=(1, 10))
        print(f"eps={eps} {name}", stats(o, b), f"{time.time() - t:.1f}s")
