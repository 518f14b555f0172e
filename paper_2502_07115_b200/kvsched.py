"""ctypes binding of libkvsched.so (include/kvsched.h) -- argument marshalling only.

Every step of the simulation runs in the CUDA kernels behind the C ABI; this module only
builds the C structs from torch tensors (device memory, streams) or numpy arrays (host
path) and turns return codes into exceptions.  There is no CPU fallback: if the library
is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libkvsched.so"

MCSF, MC_BENCH, ALPHA, ALPHA_BETA, MCSF_PROTECTED, MCSF_PROTECTED_RAISE = 0, 1, 2, 3, 4, 5
POLICY_IDS = {"mcsf": MCSF, "mcbench": MC_BENCH, "alpha": ALPHA, "alpha_beta": ALPHA_BETA,
              "mcsf_protected": MCSF_PROTECTED, "mcsf_protected_raise": MCSF_PROTECTED_RAISE}
INST_OK, INST_INVALID, INST_LIVELOCK, INST_UNSUPPORTED = 0, 1, 2, 3
FLAG_PER_ROUND = 1
FLAG_WARP_PER_INSTANCE = 2
REQ_I32X4, REQ_U16X4_DELTA, REQ_U8X4_DELTA, REQ_P16 = 0, 1, 2, 3
ERRORS = {-1: "SCHED_E_ARG", -2: "SCHED_E_CUDA", -3: "SCHED_E_NOMEM", -4: "SCHED_E_STATE"}

# every symbol include/kvsched.h declares
EXPORTS = ("sched_abi_version", "sched_init", "sched_set_stream", "sched_run_instances",
           "sched_run_instances_host", "sched_latency", "sched_lb_sorted", "sched_gen_am2_count",
           "sched_gen_am2_fill", "sched_wallclock", "sched_philox4x32_10",
           "sched_set_timing",
           "sched_get_stats", "sched_get_kernel_stats", "sched_reset_stats", "sched_last_kernel",
           "sched_finalize",
           "sched_last_error")

P = ctypes.c_void_p
i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64


class SchedInstances(ctypes.Structure):
    _fields_ = [("n_instances", i64), ("req_offset", P), ("req", P), ("mem_limit", P),
                ("instance_id0", i64), ("max_requests", i32), ("max_mem", i32),
                ("max_len", i32), ("req_format", i32)]


class SchedPolicy(ctypes.Structure):
    _fields_ = [("policy", i32), ("alpha_num", i32), ("alpha_den", i32), ("flags", i32),
                ("beta_thresh", u64), ("seed", u64), ("round_cap", i64)]


class SchedGenAm2(ctypes.Structure):
    _fields_ = [("n_instances", i64), ("instance_id0", i64), ("seed", u64), ("n_lambda", i32),
                ("n_m", i32), ("poisson_cdf", P), ("m_values", P), ("T_lo", i32), ("T_hi", i32),
                ("s_lo", i32), ("s_hi", i32)]


class SchedClock(ctypes.Structure):
    _fields_ = [("c0", i64), ("c1", i64), ("bin_width", i64), ("n_bins", i32), ("trace_len", i32)]


class SchedOutputs(ctypes.Structure):
    _fields_ = [("completion", P), ("start", P), ("tel", P), ("rounds", P),
                ("decision_rounds", P), ("evictions", P), ("makespan", P), ("peak_mem", P),
                ("status", P), ("latency16", P)]


OUT_FIELDS = ("completion", "start", "tel", "rounds", "decision_rounds", "evictions", "makespan",
              "peak_mem", "status")
OUT_I64 = ("tel", "rounds", "decision_rounds", "evictions")

_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        import os
        path = Path(os.environ.get("KVSCHED_LIB", LIB_PATH))   # experiments only
        if not path.exists():
            raise RuntimeError(f"{path} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(str(path))
        L.sched_abi_version.restype = ctypes.c_int
        L.sched_init.argtypes = [ctypes.POINTER(P), ctypes.c_int, P]
        L.sched_set_stream.argtypes = [P, P]
        for f in (L.sched_run_instances, L.sched_run_instances_host):
            f.argtypes = [P, ctypes.POINTER(SchedInstances), ctypes.POINTER(SchedPolicy),
                          ctypes.POINTER(SchedOutputs)]
        L.sched_latency.argtypes = [P, ctypes.POINTER(SchedInstances), P, P, P]
        L.sched_philox4x32_10.argtypes = [P, i64, P, P, P]
        L.sched_lb_sorted.argtypes = [P, ctypes.POINTER(SchedInstances), P]
        L.sched_gen_am2_count.argtypes = [P, ctypes.POINTER(SchedGenAm2), P]
        L.sched_wallclock.argtypes = [P, ctypes.POINTER(SchedInstances), P, P, ctypes.POINTER(SchedClock),
                                      P, P, P, P]
        L.sched_gen_am2_fill.argtypes = [P, ctypes.POINTER(SchedGenAm2), P, P, P]
        L.sched_set_timing.argtypes = [P, ctypes.c_int]
        L.sched_get_stats.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(i64)]
        L.sched_get_kernel_stats.argtypes = [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_char_p),
                                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        L.sched_reset_stats.argtypes = [P]
        L.sched_last_kernel.argtypes = [P]
        L.sched_last_kernel.restype = ctypes.c_char_p
        L.sched_finalize.argtypes = [P]
        L.sched_last_error.argtypes = [P]
        L.sched_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


@dataclass
class Policy:
    """Policy parameters as the C ABI wants them (integers only)."""
    kind: str = "mcsf"
    alpha: tuple[int, int] = (0, 1)
    beta_thresh: int = 0
    seed: int = 0
    round_cap: int = 0
    flags: int = 0            # FLAG_PER_ROUND: one round per loop iteration (A/B runs)

    def as_c(self) -> SchedPolicy:
        return SchedPolicy(POLICY_IDS[self.kind], int(self.alpha[0]), int(self.alpha[1]), int(self.flags),
                           int(self.beta_thresh), int(self.seed) & (2**64 - 1), int(self.round_cap))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class Context:
    """A library context bound to one CUDA device and (by default) torch's current stream."""

    def __init__(self, device: int = 0, stream=None):
        L = load()
        self._lib = L
        self.device = device
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(device).cuda_stream
        h = P()
        rc = L.sched_init(ctypes.byref(h), int(device), P(stream))
        if rc != 0:
            raise RuntimeError(f"sched_init: {ERRORS.get(rc, rc)}: {L.sched_last_error(None).decode()}")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sched_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != 0:
            msg = self._lib.sched_last_error(self._h).decode()
            raise RuntimeError(f"{what}: {ERRORS.get(rc, rc)}: {msg}")

    def set_stream(self, stream):
        self._check(self._lib.sched_set_stream(self._h, P(stream)), "sched_set_stream")

    # -- device path -------------------------------------------------------------------
    @staticmethod
    def instances(offset, req, mem, id0: int = 0, hints=(0, 0, 0), req_format: int = 0) -> SchedInstances:
        n = int(mem.shape[0])
        return SchedInstances(n, _ptr(offset), _ptr(req), _ptr(mem), int(id0), int(hints[0]),
                              int(hints[1]), int(hints[2]), int(req_format))

    def run(self, offset, req, mem, policy: Policy, outputs: dict, id0: int = 0,
            hints=(0, 0, 0), req_format: int = 0) -> None:
        """sched_run_instances on device tensors; `outputs` maps OUT_FIELDS names to
        preallocated device tensors (missing = not requested)."""
        si = self.instances(offset, req, mem, id0, hints, req_format)
        so = SchedOutputs(*[_ptr(outputs.get(k)) for k in OUT_FIELDS + ("latency16",)])
        pc = policy.as_c()
        self._check(self._lib.sched_run_instances(self._h, ctypes.byref(si), ctypes.byref(pc),
                                                  ctypes.byref(so)), "sched_run_instances")

    def run_host(self, offset: np.ndarray, req: np.ndarray, mem: np.ndarray, policy: Policy,
                 outputs: dict, id0: int = 0, hints=(0, 0, 0), req_format: int = 0) -> None:
        """sched_run_instances_host on host (numpy, ideally pinned) arrays."""
        si = self.instances(offset, req, mem, id0, hints, req_format)
        so = SchedOutputs(*[_ptr(outputs.get(k)) for k in OUT_FIELDS + ("latency16",)])
        pc = policy.as_c()
        self._check(self._lib.sched_run_instances_host(self._h, ctypes.byref(si), ctypes.byref(pc),
                                                       ctypes.byref(so)), "sched_run_instances_host")

    def latency(self, offset, req, completion, tel=None, tel_total=None) -> None:
        n = int(offset.shape[0]) - 1
        si = SchedInstances(n, _ptr(offset), _ptr(req), None, 0, 0, 0, 0, 0)
        self._check(self._lib.sched_latency(self._h, ctypes.byref(si), _ptr(completion), _ptr(tel),
                                            _ptr(tel_total)), "sched_latency")

    def lb_sorted(self, offset, req, mem, lb, hints=(0, 0, 0)) -> None:
        """sched_lb_sorted: lb[k] = volume lower bound on OPT of simultaneous-arrival instances."""
        si = self.instances(offset, req, mem, 0, hints)
        self._check(self._lib.sched_lb_sorted(self._h, ctypes.byref(si), _ptr(lb)), "sched_lb_sorted")

    def wallclock(self, offset, req, mem, start, completion, c0: int, c1: int, bin_width: int = 0,
                  n_bins: int = 0, trace_len: int = 0) -> dict:
        """NEXT-4: wall clock of a schedule (sched_wallclock); returns device tensors."""
        import torch
        dev = start.device
        n = int(offset.shape[0]) - 1
        out = dict(tel_wall=torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                   makespan_wall=torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                   bins=torch.empty((max(n, 1), max(n_bins, 1)), dtype=torch.int64, device=dev),
                   mem=torch.empty((max(n, 1), max(trace_len, 1)), dtype=torch.int32, device=dev))
        si = self.instances(offset, req, mem)
        ck = SchedClock(int(c0), int(c1), int(bin_width), int(n_bins), int(trace_len))
        self._check(self._lib.sched_wallclock(self._h, ctypes.byref(si), _ptr(start), _ptr(completion), ctypes.byref(ck),
                                              _ptr(out["tel_wall"]), _ptr(out["makespan_wall"]),
                                              _ptr(out["bins"]) if n_bins else None,
                                              _ptr(out["mem"]) if trace_len else None), "sched_wallclock")
        return out

    def gen_am2(self, n_inst: int, spec, id0: int = 0):
        """NEXT-3: generate an AM2-grid batch on the device (sched_gen_am2_count + _fill).
        `spec` is a workloads.Am2Spec; returns device tensors (offset, req, mem)."""
        import torch
        dev = torch.device("cuda", self.device)
        cdf = torch.from_numpy(spec.tables().astype(np.uint64).view(np.int64)).to(dev)
        ms = torch.tensor(list(spec.Ms), dtype=torch.int32, device=dev)
        g = SchedGenAm2(int(n_inst), int(id0), int(spec.seed) & (2**64 - 1), len(spec.lambdas), len(spec.Ms),
                        cdf.data_ptr(), ms.data_ptr(), int(spec.T_lo), int(spec.T_hi), int(spec.s_lo),
                        int(spec.s_hi))
        off = torch.empty(int(n_inst) + 1, dtype=torch.int64, device=dev)
        self._check(self._lib.sched_gen_am2_count(self._h, ctypes.byref(g), off.data_ptr()), "sched_gen_am2_count")
        n_req = int(off[-1].item())                      # one 8-byte read to size the rows
        req = torch.empty((max(n_req, 1), 4), dtype=torch.int32, device=dev)
        mem = torch.empty(max(int(n_inst), 1), dtype=torch.int32, device=dev)
        self._check(self._lib.sched_gen_am2_fill(self._h, ctypes.byref(g), off.data_ptr(), req.data_ptr(),
                                                 mem.data_ptr()), "sched_gen_am2_fill")
        return off, req[:max(n_req, 1)], mem[:max(int(n_inst), 1)], n_req

    def philox(self, ctr, key, out) -> None:
        n = int(ctr.shape[0])
        self._check(self._lib.sched_philox4x32_10(self._h, n, _ptr(ctr), _ptr(key), _ptr(out)),
                    "sched_philox4x32_10")

    # -- accounting ----------------------------------------------------------------------
    def set_timing(self, on: bool = True):
        self._check(self._lib.sched_set_timing(self._h, 1 if on else 0), "sched_set_timing")

    def stats(self) -> dict:
        a, b, c = i64(), ctypes.c_double(), i64()
        self._check(self._lib.sched_get_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
                    "sched_get_stats")
        return dict(launches=a.value, sim_kernel_ms=b.value, sim_kernel_launches=c.value)

    def kernel_stats(self) -> dict:
        """{kernel name: (device ms, launches)} since the last reset (timing enabled)."""
        out, i = {}, 0
        while True:
            nm, ms, n = ctypes.c_char_p(), ctypes.c_double(), i64()
            if self._lib.sched_get_kernel_stats(self._h, i, ctypes.byref(nm), ctypes.byref(ms), ctypes.byref(n)):
                return out
            out[nm.value.decode()] = (ms.value, n.value)
            i += 1

    def reset_stats(self):
        self._check(self._lib.sched_reset_stats(self._h), "sched_reset_stats")

    def last_kernel(self) -> str:
        return self._lib.sched_last_kernel(self._h).decode()


# ---------------------------------------------------------------------------------------
# convenience: allocate outputs with torch and run a workloads.Batch-like object
# ---------------------------------------------------------------------------------------
def alloc_outputs(n_inst: int, n_req: int, device, fields=OUT_FIELDS) -> dict:
    import torch
    out = {}
    for k in fields:
        if k in ("completion", "start"):
            out[k] = torch.empty(max(n_req, 1), dtype=torch.int32, device=device)
        elif k in OUT_I64:
            out[k] = torch.empty(max(n_inst, 1), dtype=torch.int64, device=device)
        else:
            out[k] = torch.empty(max(n_inst, 1), dtype=torch.int32, device=device)
    return out


def to_device(batch, device):
    """(offset, req, mem) torch tensors on `device` from a host batch."""
    import torch
    off = torch.from_numpy(np.ascontiguousarray(batch.offset)).to(device)
    req = torch.from_numpy(np.ascontiguousarray(batch.req)).to(device)
    if req.numel() == 0:
        req = torch.zeros((1, 4), dtype=torch.int32, device=device)
    mem = torch.from_numpy(np.ascontiguousarray(batch.mem)).to(device)
    return off, req, mem


def hints_of(batch) -> tuple[int, int, int]:
    return (max(batch.max_requests(), 1), max(batch.max_mem(), 1), max(batch.max_len(), 1))


def simulate(ctx: Context, batch, policy: Policy, id0: int = 0, hints=None, fields=OUT_FIELDS,
             packed=False, latency16: bool = False) -> dict:
    """Run a host batch on the device; returns numpy arrays trimmed to the batch size.
    packed=True / "u16" ships the rows as SCHED_REQ_U16X4_DELTA, "u8" as SCHED_REQ_U8X4_DELTA,
    "p16" as SCHED_REQ_P16 (decoded on the device); latency16=True also requests the compact uint16 schedule."""
    import torch
    dev = torch.device("cuda", ctx.device)
    off, req, mem = to_device(batch, dev)
    fmt = REQ_I32X4
    if packed:
        pk = {"u8": batch.packed_u8, "p16": batch.packed_p16}.get(packed, batch.packed_u16)()
        if pk is None:
            raise ValueError(f"batch does not fit the {packed} encoding")
        dt = np.int8 if packed == "u8" else np.int16
        req = torch.from_numpy(pk.view(dt) if pk.size else np.zeros((1, 4), dt)).to(dev)
        fmt = {"u8": REQ_U8X4_DELTA, "p16": REQ_P16}.get(packed, REQ_U16X4_DELTA)
    out = alloc_outputs(batch.n_inst, batch.n_req, dev, fields)
    if latency16:
        out["latency16"] = torch.empty(max(batch.n_req, 1), dtype=torch.int16, device=dev)
    ctx.run(off, req, mem, policy, out, id0=id0, hints=hints if hints is not None else (0, 0, 0),
            req_format=fmt)
    torch.cuda.synchronize(dev)
    res = {}
    for k, v in out.items():
        n = batch.n_inst if k not in ("completion", "start", "latency16") else batch.n_req
        a = v.cpu().numpy()[:n]
        res[k] = a.view(np.uint16) if k == "latency16" else a
    return res
