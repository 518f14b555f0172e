"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (CPU, -m "not gpu").

oracle/oracle.c is compiled together with tests/native/oracle_san_driver.c with
-fsanitize=address,undefined and run over seeded batches of every shape the tests use
(ragged, empty instances, the lane kernel's scope edges, trace-shaped, prediction noise)
for all five policies.  Any sanitizer report fails the run (halt_on_error); the outputs must
also equal the regular -O2 build's, so the sanitized build checks the same code.
"""
import os
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import workloads as W

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def san_driver(tmp_path_factory):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    out = tmp_path_factory.mktemp("san") / "oracle_san"
    cmd = ["gcc", "-O1", "-g", "-std=gnu11", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
           "-fno-sanitize-recover=all", str(ROOT / "oracle" / "oracle.c"),
           str(ROOT / "tests" / "native" / "oracle_san_driver.c"), "-o", str(out), "-lpthread"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def _write(path, b):
    with open(path, "wb") as f:
        np.array([b.n_inst], np.int64).tofile(f)
        np.asarray(b.offset, np.int64).tofile(f)
        np.ascontiguousarray(b.req, np.int32).tofile(f)
        np.asarray(b.mem, np.int32).tofile(f)


BATCHES = {
    "ragged": lambda: W.random_small(300, 61, n_max=40, M_lo=4, M_hi=120, a_max=40),
    "lane_edges": lambda: W.lane_mix(200, 62, n_max=130, s_max=9, gap_max=600),
    "trace": lambda: W.c4(3, 63),
    "noisy": lambda: W.with_prediction_noise(W.random_small(200, 64, n_max=25, M_lo=10, M_hi=60, a_max=20), 0.8),
    "c1": lambda: W.c1(300, 65, "b"),
}
POLICIES = [(0, (0, 1), 0, 0), (1, (0, 1), 0, 0), (2, (1, 10), 0, 0), (3, (1, 5), 2**31, 9), (4, (1, 10), 0, 0)]


@pytest.mark.parametrize("name", list(BATCHES))
@pytest.mark.parametrize("pol,alpha,beta,seed", POLICIES, ids=["mcsf", "mcbench", "alpha", "alpha_beta", "prot"])
def test_oracle_clean_under_asan_ubsan(san_driver, oracle_mod, tmp_path, name, pol, alpha, beta, seed):
    b = BATCHES[name]()
    src, dst = tmp_path / "batch.bin", tmp_path / "out.bin"
    _write(src, b)
    env = dict(os.environ, ASAN_OPTIONS="halt_on_error=1:detect_leaks=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    r = subprocess.run([str(san_driver), str(src), str(pol), str(alpha[0]), str(alpha[1]), str(beta),
                        str(seed), str(dst)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "runtime error" not in r.stderr and "Sanitizer" not in r.stderr, r.stderr[-3000:]
    raw = dst.read_bytes()
    nr, ni = b.n_req, b.n_inst
    comp = np.frombuffer(raw, np.int32, nr, 0)
    start = np.frombuffer(raw, np.int32, nr, 4 * nr)
    stats = np.frombuffer(raw, np.int64, 7 * ni, 8 * nr).reshape(ni, 7)
    o = oracle_mod.simulate_batch(b.offset, b.req, b.mem, pol, alpha=alpha, beta_thresh=beta, seed=seed)
    assert np.array_equal(comp, o["completion"]) and np.array_equal(start, o["start"])
    for j, k in enumerate(("tel", "rounds", "decision_rounds", "makespan", "peak", "evictions", "status")):
        assert np.array_equal(stats[:, j], np.asarray(o[k], np.int64)), k
