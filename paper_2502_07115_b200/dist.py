"""Multi-GPU plumbing: instance sharding and the result exchange (torch.distributed).

Instances are independent (one worker per instance), so the path shards with no
data-path collective.  The only exchange is the one the north star names: every rank gathers
the per-instance (TEL, rounds, status) of all shards and all ranks reduce the totals.  With
the NCCL backend these run over NVLink/NVSwitch; the same code runs on gloo (CPU tests).

Shard k of W covers global instances [lo_k, hi_k); its `instance_id0` is lo_k, which also
keys the alpha-beta RNG, so outputs do not depend on how a batch is split.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

RESULT_ROWS = ("tel", "rounds", "status")


def shard_bounds(n_total: int, world: int, rank: int, weights=None) -> tuple[int, int]:
    """Contiguous shard of [0, n_total) for `rank`.  With per-instance `weights` (e.g. the
    request counts) the cut points balance the summed weight, else the instance count."""
    if world <= 1:
        return 0, n_total
    if weights is None:
        base, extra = divmod(n_total, world)
        lo = rank * base + min(rank, extra)
        return lo, lo + base + (1 if rank < extra else 0)
    w = torch.as_tensor(weights, dtype=torch.float64)
    cum = torch.cumsum(w, 0)
    total = float(cum[-1]) if n_total else 0.0

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return n_total
        return int(torch.searchsorted(cum, torch.tensor(total * r / world, dtype=torch.float64)).item())
    return cut(rank), cut(rank + 1)


def result_dtype(batch, policy: str = "mcsf", round_cap: int = 0) -> torch.dtype:
    """int32 rows when every TEL and round count provably fits, else int64.  Halves the bytes
    the gather moves on the bench workloads.

    Bounds (per instance, n requests, c_i the completion of an OK run):
      MC-SF / MC-Benchmark: every round with S empty admits the head, so c_i <= max_a + sum o
        and TEL <= n (max_a + sum o);
      evicting policies (alpha, alpha-beta, protected MC-SF): a run can last until the round
        cap, so c_i <= cap + max o <= cap + sum o, cap = round_cap if > 0 else the default
        min(2^30, 16 (max_a + sum o) + 64) (DESIGN Q23), and TEL <= n (cap + sum o)."""
    import numpy as np
    if batch.n_inst == 0 or batch.n_req == 0:
        return torch.int32
    sizes = np.diff(batch.offset)
    last = batch.offset[1:] - 1
    amax = np.where(sizes > 0, batch.req[np.maximum(last, 0), 0].astype(np.int64), 0)
    sumo = np.add.reduceat(batch.req[:, 2].astype(np.int64), np.minimum(batch.offset[:-1], batch.n_req - 1))
    sumo = np.where(sizes > 0, sumo, 0)
    if policy in ("mcsf", "mcbench"):
        horizon = amax + sumo
    else:
        cap = np.full_like(amax, int(round_cap)) if round_cap > 0 else \
            np.minimum(16 * (amax + sumo) + 64, 2 ** 30)
        horizon = cap + sumo
    bound = int((sizes * horizon).max(initial=0))
    return torch.int32 if bound < 2**31 - 1 else torch.int64


def pack_results(out: dict, n_local: int, n_pad: int, device, dtype=torch.int64) -> torch.Tensor:
    """[3, n_pad] rows (TEL, rounds, status) of this shard, padded with status -1."""
    buf = torch.full((len(RESULT_ROWS), n_pad), -1, dtype=dtype, device=device)
    for i, k in enumerate(RESULT_ROWS):
        buf[i, :n_local].copy_(out[k][:n_local])
    return buf


def gather_results(local: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of the [3, n_pad] shard rows -> [world, 3, n_pad]."""
    world = dist.get_world_size(group)
    out = torch.empty((world, *local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    elif local.is_cuda:                 # gloo: through host memory (multi-rank tests on one GPU)
        parts = [torch.empty(local.shape, dtype=local.dtype) for _ in range(world)]
        dist.all_gather(parts, local.cpu().contiguous(), group=group)
        out.copy_(torch.stack(parts))
    else:
        dist.all_gather(list(out.unbind(0)), local.contiguous(), group=group)
    return out


def reduce_totals(out: dict, n_local: int, group=None) -> torch.Tensor:
    """all_reduce(SUM) of [sum TEL, sum rounds, #OK, #instances] over OK instances
    (integer sums: exact in any reduction order)."""
    ok = out["status"][:n_local] == 0
    tot = torch.stack([
        torch.where(ok, out["tel"][:n_local], torch.zeros_like(out["tel"][:n_local])).sum(),
        torch.where(ok, out["rounds"][:n_local], torch.zeros_like(out["rounds"][:n_local])).sum(),
        ok.sum().to(torch.int64),
        torch.full((), n_local, dtype=torch.int64, device=ok.device),   # a fill, no host copy
    ])
    if dist.is_initialized():
        dist.all_reduce(tot, group=group)
    return tot


def unpad(gathered: torch.Tensor, sizes) -> torch.Tensor:
    """[world, 3, n_pad] -> [3, sum(sizes)] in global instance order."""
    parts = [gathered[r, :, :int(n)] for r, n in enumerate(sizes)]
    return torch.cat(parts, dim=1)
