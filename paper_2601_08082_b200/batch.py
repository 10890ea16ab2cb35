"""Batched and multi-GPU drivers for independent SPD systems (BASELINE
config C4: 64 x N=16384 POTRF + POTRS).

The path shards naturally: systems are independent, so a batch is split
across ranks (one process per GPU, ``torch.distributed``) with NO data-path
collective.  Each rank factors and solves its own contiguous share on its
own device through :class:`paper_2601_08082_b200.Batch` (several plans side
by side); the only communication is the final reduction of per-rank
counters and the max-over-ranks device time.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


def shard(count: int, world: int, rank: int) -> range:
    """contiguous share of `count` systems for `rank` (sizes differ by <= 1)"""
    if world < 1 or not 0 <= rank < world or count < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(count, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class ShardResult:
    systems: int          # systems this rank factored
    failed: int           # systems whose status was not ok
    device_ms: float      # this rank's device time (max over ranks after reduce)
    worst_residual: float  # max ||b - A x|| / (||A||_F ||x|| + ||b||) over the checked systems
    solve_ms: float = 0.0  # device time of the batched solve phases (max over ranks after reduce)


def reduce_results(local: ShardResult, group=None) -> ShardResult:
    """sum systems / failures, max time and residual over ranks (host-side
    bookkeeping only; works on gloo and nccl)"""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    s = torch.tensor([float(local.systems), float(local.failed)], dtype=torch.float64, device=dev)
    m = torch.tensor([local.device_ms, local.worst_residual if math.isfinite(local.worst_residual) else 1e300,
                      local.solve_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    return ShardResult(int(s[0].item()), int(s[1].item()), float(m[0].item()), float(m[1].item()),
                       float(m[2].item()))


def spd_generate_many(n: int, seeds, device="cuda", threads: int = 0):
    """spd_generate(n, seed) for every seed, bit-identical (analysis.cpp:12-28),
    straight into device tensors.  The mt19937_64 draw stream is sequential per
    matrix, so matrices are generated side by side on host threads (the C
    call releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import paper_2601_08082_b200 as tc
    seeds = list(seeds)
    if not seeds:
        return []
    threads = threads or min(len(seeds), max(1, (os.cpu_count() or 2) // 2), 16)
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda sd: tc.spd_generate_device(n, sd, device), seeds))


def synthetic_spd_device(n: int, seed: int, device="cuda"):
    """device-generated SPD matrix of spd_generate's distribution
    (analysis.cpp:12-28: symmetrized uniform [0,1), n added to the diagonal),
    column-major (to_device layout).  Fast on the GPU, not bit-identical to the
    mt19937_64 stream -- throughput runs only; parity uses spd_generate."""
    import torch
    g = torch.Generator(device=device).manual_seed(int(seed))
    r = torch.rand((n, n), dtype=torch.float64, device=device, generator=g)
    a = (r + r.T).mul_(0.5)
    a.diagonal().add_(float(n))
    return a


def run_batch_on_rank(count: int, n: int, b: int, config, seed0: int = 0, nrhs: int = 1, concurrency: int = 8,
                      world: int = 1, rank: int = 0, group=None, check: int = 1, in_flight: int = 16,
                      options: dict | None = None):
    """factor + solve this rank's share of a batch of `count` systems
    A_k = spd_generate(n, seed0 + k) (bit-identical), b_k = A_k * ones.
    Returns (local ShardResult, reduced ShardResult, flops per system)."""
    import torch
    import paper_2601_08082_b200 as tc
    mine = shard(count, world, rank)
    batch = tc.Batch(n, b, config, True, concurrency)
    for k, v in (options or {}).items():
        batch.set_option(k, v)
    # warm-up (untimed): builds every plan's workspace and CUDA graph, and
    # sizes the per-call buffers (status words, POTRS workspace and pointer
    # tables) for in_flight systems, so no allocation lands in a timed call
    warm = [synthetic_spd_device(n, seed0 + 10 ** 6 + k) for k in range(concurrency)]
    warm += [warm[k % concurrency].clone() for k in range(concurrency, min(in_flight, len(mine)))]
    wb = [a.sum(dim=0, keepdim=True).repeat(nrhs, 1).contiguous() for a in warm]
    batch.run(warm, wb)  # the solve path too (its workspace, first kernel loads)
    del warm, wb
    torch.cuda.synchronize()
    failed, worst, dev_ms, solve_ms = 0, 0.0, 0.0, 0.0
    ks = list(mine)
    for c0 in range(0, len(ks), in_flight):
        chunk = ks[c0:c0 + in_flight]
        a_list = spd_generate_many(n, [seed0 + k for k in chunk])
        keep = [a.clone() for a in a_list[:check]] if c0 == 0 else []
        # right-hand sides b = A * 1 (x_true = ones), column-major (nrhs, n)
        b_list = [a.sum(dim=0, keepdim=True).repeat(nrhs, 1).contiguous() for a in a_list]
        rhs0 = [x.clone() for x in b_list[:len(keep)]]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = batch.run(a_list, b_list)
        e1.record()
        torch.cuda.synchronize()
        dev_ms += e0.elapsed_time(e1)
        solve_ms += batch.last_solve_ms()
        failed += sum(1 for x in st if x != "ok")
        for a0, x, b0 in zip(keep, b_list, rhs0):
            worst = max(worst, tc.solve_residual_device(a0, x[0].contiguous(), b0[0].contiguous()))
        del a_list, b_list, keep, rhs0
    local = ShardResult(len(ks), failed, dev_ms, worst, solve_ms)
    flops = tc.potrf_flops(n) + 2 * n * n * nrhs
    return local, reduce_results(local, group), flops
