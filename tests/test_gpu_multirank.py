"""The bench's N > 1 path (torchrun, one process per rank) against its 1-rank run.

The box has one GPU, so both ranks share cuda:0 and talk over gloo (KVSCHED_BENCH_ONE_GPU /
KVSCHED_BENCH_BACKEND: the code path of an 8-GPU NCCL run minus the transport).  With the
strong split the ranks cut the config's batch by dist.shard_bounds (weighted by request
count) and key their instances by global id, so the gathered per-instance (TEL, rounds,
status) rows must equal the 1-rank run's byte for byte (SURVEY 8(e) shard invariance).
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(tmp, nproc, extra, name, e2e=False):
    dump = tmp / f"{name}.npy"
    args = ["bench.py", "--gpus", str(nproc), "--steps", "2", "--warmup", "3", "--no-also",
            "--no-cpu-baseline", "--dump-results", str(dump), *extra]
    if not e2e:
        args.append("--no-e2e")
    env = dict(os.environ, KVSCHED_BENCH_ONE_GPU="1", KVSCHED_BENCH_BACKEND="gloo")
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), *args]
    else:
        cmd = [sys.executable, *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return lines[0], np.load(dump)


@pytest.mark.parametrize("extra", [["--workload", "c5", "--instances", "30000"],
                                   ["--workload", "c4", "--instances", "600", "--policy", "alpha_beta"],
                                   ["--workload", "c4", "--instances", "600", "--policy", "mcsf"]],
                         ids=["c5-mcsf", "c4-alpha-beta", "c4-mcsf"])
def test_strong_split_equals_one_rank(tmp_path, extra):
    one, r1 = _bench(tmp_path, 1, extra, "one")
    for n in (2, 3):
        line, rn = _bench(tmp_path, n, extra, f"n{n}")
        assert line["n_gpus"] == n and line["scaling"] == "strong"
        assert line["config"]["instances_total"] == one["config"]["instances_total"]
        assert rn.dtype == r1.dtype and rn.shape == r1.shape
        assert np.array_equal(rn, r1), f"{n} ranks differ from 1 rank"
        assert line["config"]["rounds_per_step"] == one["config"]["rounds_per_step"]


def test_weak_split_runs_every_rank(tmp_path):
    extra = ["--workload", "c5", "--instances", "5000", "--split", "weak"]
    one, r1 = _bench(tmp_path, 1, extra, "one")
    line, r2 = _bench(tmp_path, 2, extra, "two")
    assert line["scaling"] == "weak" and line["config"]["instances_total"] == 10_000
    assert r2.shape[1] == 10_000 and np.array_equal(r2[:, :5000], r1)


def test_streamed_host_path_per_rank(tmp_path):
    """The e2e leg at N > 1: every rank runs its shard through sched_run_instances_host (P16
    rows: the streamed pipeline) and checks it against its device-path run
    (matches_device_run); rank 0 reports, the gathered device results equal the 1-rank run."""
    extra = ["--workload", "c5", "--instances", "20000", "--e2e-steps", "2"]
    one, r1 = _bench(tmp_path, 1, extra, "one", e2e=True)
    assert one["e2e"]["matches_device_run"] and one["e2e"]["req_format"] == "p16"
    line, r2 = _bench(tmp_path, 2, extra, "two", e2e=True)
    assert line["e2e"]["matches_device_run"]
    assert np.array_equal(r2, r1)
