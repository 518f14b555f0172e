"""Multi-process (gloo, world size 2, CPU) tests of the sharding and result exchange.

Each rank takes its shard of a batch, computes that shard's per-instance results (here with
the CPU oracle: the host-side exchange logic is what is under test), and the gathered /
reduced results must equal the whole-batch run.  The alpha-beta RNG is keyed by the global
instance id, so the shard results themselves must not depend on the split either.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2502_07115_b200 import dist as D
        b = W.random_small(301, 7, n_max=30, M_lo=10, M_hi=60, a_max=20)
        sizes = [D.shard_bounds(b.n_inst, world, r, weights=b.sizes())[1] -
                 D.shard_bounds(b.n_inst, world, r, weights=b.sizes())[0] for r in range(world)]
        lo, hi = D.shard_bounds(b.n_inst, world, rank, weights=b.sizes())
        sub = b.subset(range(lo, hi))
        o = oracle.simulate_batch(sub.offset, sub.req, sub.mem, oracle.ALPHA_BETA, alpha=(1, 10),
                                  beta_thresh=W.beta_threshold(0.3), seed=11, gid0=lo, nthreads=1)
        out = {k: torch.from_numpy(np.asarray(o[k], dtype=np.int64)) for k in ("tel", "rounds", "status")}
        local = D.pack_results(out, hi - lo, max(sizes), "cpu", D.result_dtype(sub))
        g = D.gather_results(local)
        tot = D.reduce_totals(out, hi - lo)
        if rank == 0:
            q.put((D.unpad(g, sizes).numpy(), tot.numpy(), sizes))
    finally:
        dist.destroy_process_group()


def test_shard_bounds():
    from paper_2502_07115_b200 import dist as D
    for n, w in ((10, 3), (0, 2), (7, 8), (1000, 8)):
        cuts = [D.shard_bounds(n, w, r) for r in range(w)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        assert all(cuts[r][1] == cuts[r + 1][0] for r in range(w - 1))
        assert max(b - a for a, b in cuts) - min(b - a for a, b in cuts) <= 1
    wts = np.array([1] * 90 + [100] * 10)
    cuts = [D.shard_bounds(100, 2, r, weights=wts) for r in range(2)]
    assert cuts[0][1] < 95 and cuts[0][0] == 0 and cuts[1][1] == 100


def test_gloo_world2_gather_equals_whole_batch():
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, tot, sizes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b = W.random_small(301, 7, n_max=30, M_lo=10, M_hi=60, a_max=20)
    whole = oracle.simulate_batch(b.offset, b.req, b.mem, oracle.ALPHA_BETA, alpha=(1, 10),
                                  beta_thresh=W.beta_threshold(0.3), seed=11, gid0=0)
    assert sum(sizes) == b.n_inst and min(sizes) > 0
    assert np.array_equal(rows[0], whole["tel"])
    assert np.array_equal(rows[1], whole["rounds"])
    assert np.array_equal(rows[2], whole["status"])
    ok = whole["status"] == 0
    assert tot.tolist() == [int(whole["tel"][ok].sum()), int(whole["rounds"][ok].sum()), int(ok.sum()), b.n_inst]


def test_result_dtype_bound():
    from paper_2502_07115_b200 import dist as D
    assert D.result_dtype(W.am2(200, 3)) == torch.int32
    big = W.from_instances([([[0, 1, 30000, 30000]] * 80000, 2**20)])
    assert D.result_dtype(big) == torch.int64
    assert D.result_dtype(W.from_instances([([], 7)])) == torch.int32
    # MC bound n (max_a + sum o) = 2000 * 1e6 fits int32; an evicting policy may run to the
    # round cap 16x later, whose bound does not (no silent wrap in the gather)
    mid = W.from_instances([([[0, 1, 500, 500]] * 2000, 1002)])
    assert D.result_dtype(mid, "mcsf") == torch.int32
    for pol in ("alpha", "alpha_beta", "mcsf_protected"):
        assert D.result_dtype(mid, pol) == torch.int64
    assert D.result_dtype(mid, "alpha", round_cap=1000) == torch.int32


def test_bench_strong_split_partitions_the_config_batch():
    """bench.make_workload(split="strong"): the shards of ranks 0..W-1 are contiguous,
    cover the config's batch exactly once, carry their global first id, and are balanced by
    request count."""
    import bench
    full, _ = bench.make_workload("c4", 300, 0)
    full = full[0]
    for world in (2, 3, 8):
        parts = [bench.make_workload("c4", 300, r, world, "strong") for r in range(world)]
        ids = [p[0][1] for p in parts]
        sizes = [p[0][0].n_inst for p in parts]
        assert ids == [sum(sizes[:r]) for r in range(world)] and sum(sizes) == full.n_inst
        req = np.concatenate([p[0][0].req for p in parts])
        assert np.array_equal(req, full.req)
        assert parts[0][1]["shard_sizes"] == sizes
        nreq = [p[0][0].n_req for p in parts]
        assert max(nreq) - min(nreq) <= 2 * int(full.sizes().max())
