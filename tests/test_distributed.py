"""Distributed single factorization (BASELINE config C5): the top split's
TRSM and SYRK row-split over ranks, A11 / A22 factored on rank 0.

CPU: the row partitions (equal TRSM rows; SYRK rows balanced by
lower-triangle work on leaf boundaries), the level shift of depth-1
subtrees, and the memory budget of the compact pieces at the BASELINE size
(N = 131072 on 8 GPUs: every rank <= 150 GB of a B200's 180 GB; planner
only -- unmeasured on hardware).
GPU: the distributed factor equals the single-device factor BIT FOR BIT --
with one rank (no process group) and with two and four ranks sharing one GPU
over a gloo group (collectives staged through host memory).  Every block
receives the same operations in the same order; row blocks of a GEMM / TRSM
are independent, so the split changes no element's arithmetic.
"""
import os
import socket

import numpy as np
import pytest

from paper_2601_08082_b200.distributed import (leaf_starts, memory_plan, row_partition, shifted_levels,
                                               syrk_partition)

N, B, CFG, SEED = 2048, 128, "[F16, F16, F16, F32]", 5


def test_row_partition_covers_and_aligns():
    for n2, world, al in ((1024, 2, 128), (1000, 3, 64), (65536, 8, 256), (256, 4, 256)):
        parts = row_partition(n2, world, al)
        assert parts[0][0] == 0 and parts[-1][1] == n2
        for (a, b_), (c, d) in zip(parts, parts[1:]):
            assert b_ == c
        for lo, hi in parts:
            assert lo % al == 0 and (hi % al == 0 or hi == n2) and lo <= hi


def test_syrk_partition_balances_lower_triangle_work():
    for n2, b, world in ((65536, 256, 8), (1024, 128, 4), (2048, 128, 2), (1000, 64, 3), (4096, 256, 4)):
        parts = syrk_partition(n2, b, world)
        cuts = set(leaf_starts(n2, b))
        assert parts[0][0] == 0 and parts[-1][1] == n2
        for (a, b_), (c, _) in zip(parts, parts[1:]):
            assert b_ == c
        for lo, hi in parts:
            assert lo in cuts and hi in cuts and lo <= hi
        work = [hi * hi - lo * lo for lo, hi in parts]
        if n2 // b >= 8 * world:
            assert max(work) <= 1.25 * n2 * n2 / world, work


def test_c5_memory_budget_at_baseline_size():
    """BASELINE C5: N = 131072, b = 256, [F16, F16, F16, F32] on 8 GPUs --
    every rank's peak device memory (plans' workspace from the planner plus
    the operands it holds) within 150 GB (unmeasured on hardware)"""
    per_rank = memory_plan(131072, 256, "[F16, F16, F16, F32]", 8)
    assert len(per_rank) == 8
    assert max(per_rank) <= 150e9, [round(x / 1e9, 1) for x in per_rank]
    # the order-65536 subproblems dominate rank 0; the others hold only pieces
    assert max(per_rank[1:]) <= 60e9, [round(x / 1e9, 1) for x in per_rank]


def test_shifted_levels():
    assert shifted_levels((0, 0, 0, 1)) == (0, 0, 1)
    assert shifted_levels((2,)) == (2,)


def _pieces(tc, n, seed, world, rank):
    """this rank's inputs, cut from the full (column-major) matrix"""
    import torch
    a = tc.spd_generate_device(n, seed)
    n1 = n // 2
    n2 = n - n1
    lo, hi = row_partition(n2, world, B)[rank]
    slo, shi = syrk_partition(n2, B, world)[rank]
    a11 = a[:n1, :n1].contiguous() if rank == 0 else None
    l22 = torch.empty((n2, n2), dtype=torch.float64, device="cuda") if rank == 0 else None
    a21 = a[:n1, n1 + lo:n1 + hi].contiguous()      # TRSM rows n1+lo.., cols 0..n1
    a22 = a[n1:, n1 + slo:n1 + shi].contiguous()    # SYRK rows n1+slo.., cols n1..
    return a, a11, a21, a22, l22


def _single(tc, n, seed):
    import torch
    a = tc.spd_generate_device(n, seed)
    l = torch.empty_like(a)
    st = tc.Plan(n, B, CFG).factor_device(a, l)
    assert st.status == "ok"
    return l


def _lower_equal(x, y):
    x, y = x.cpu().numpy(), y.cpu().numpy()  # (cols, rows): element (i, j) at [j, i]
    return np.array_equal(np.tril(x.T), np.tril(y.T))


@pytest.mark.gpu
def test_distributed_single_rank_bit_identical(tc):
    from paper_2601_08082_b200.distributed import potrf_top_split
    ref = _single(tc, N, SEED)
    a, a11, a21, a22, l22 = _pieces(tc, N, SEED, 1, 0)
    res = potrf_top_split(N, B, CFG, a11=a11, a21_rows=a21, a22_rows=a22, l22=l22)
    assert res.status == "ok"
    n1 = N // 2
    assert _lower_equal(res.l11, ref[:n1, :n1])
    assert np.array_equal(res.l21_rows.cpu().numpy(), ref[:n1, n1:].cpu().numpy())
    assert _lower_equal(res.l22, ref[n1:, n1:])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, outdir, n=N):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2601_08082_b200 as tc
    from paper_2601_08082_b200.distributed import potrf_top_split
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, a11, a21, a22, l22 = _pieces(tc, n, SEED, world, rank)
    res = potrf_top_split(n, B, CFG, a11=a11, a21_rows=a21, a22_rows=a22, l22=l22)
    np.save(os.path.join(outdir, f"l21_{rank}.npy"), res.l21_rows.cpu().numpy())
    if rank == 0:
        np.save(os.path.join(outdir, "l11.npy"), res.l11.cpu().numpy())
        np.save(os.path.join(outdir, "l22.npy"), res.l22.cpu().numpy())
    with open(os.path.join(outdir, f"status_{rank}"), "w") as f:
        f.write(res.status)
    dist.destroy_process_group()


def _run_world(tc, tmp_path, world, n):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path), n)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=900)
        assert p.exitcode == 0
    for r in range(world):
        assert open(tmp_path / f"status_{r}").read() == "ok"
    ref = _single(tc, n, SEED).cpu().numpy()
    n1 = n // 2
    parts = row_partition(n - n1, world, B)
    assert np.array_equal(np.tril(np.load(tmp_path / "l11.npy").T), np.tril(ref[:n1, :n1].T))
    for r, (lo, hi) in enumerate(parts):
        assert np.array_equal(np.load(tmp_path / f"l21_{r}.npy"), ref[:n1, n1 + lo:n1 + hi])
    assert np.array_equal(np.tril(np.load(tmp_path / "l22.npy").T), np.tril(ref[n1:, n1:].T))


@pytest.mark.gpu
def test_distributed_two_ranks_one_gpu_bit_identical(tc, tmp_path):
    _run_world(tc, tmp_path, 2, N)


@pytest.mark.gpu
def test_distributed_four_ranks_n4096_bit_identical(tc, tmp_path):
    """the verdict's check: 4 ranks (gloo, one GPU), N = 4096"""
    _run_world(tc, tmp_path, 4, 4096)
