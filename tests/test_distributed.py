"""Distributed single factorization (BASELINE config C5): the top split's
TRSM and SYRK row-split over ranks, A11 / A22 factored on rank 0.

CPU: the row partition and the level shift of depth-1 subtrees.
GPU: the distributed factor equals the single-device factor BIT FOR BIT --
with one rank (no process group) and with two ranks sharing one GPU over a
gloo group (collectives staged through host memory).  Every block receives
the same operations in the same order; row blocks of a GEMM / TRSM are
independent, so the split changes no element's arithmetic.
"""
import os
import socket

import numpy as np
import pytest

from paper_2601_08082_b200.distributed import row_partition, shifted_levels

N, B, CFG, SEED = 2048, 128, "[F16, F16, F16, F32]", 5


def test_row_partition_covers_and_aligns():
    for n2, world, al in ((1024, 2, 128), (1000, 3, 64), (65536, 8, 256), (256, 4, 256)):
        parts = row_partition(n2, world, al)
        assert parts[0][0] == 0 and parts[-1][1] == n2
        for (a, b_), (c, d) in zip(parts, parts[1:]):
            assert b_ == c
        for lo, hi in parts:
            assert lo % al == 0 and (hi % al == 0 or hi == n2) and lo <= hi


def test_shifted_levels():
    assert shifted_levels((0, 0, 0, 1)) == (0, 0, 1)
    assert shifted_levels((2,)) == (2,)


def _pieces(tc, n, seed, world, rank):
    """this rank's inputs, cut from the full (column-major) matrix"""
    a = tc.spd_generate_device(n, seed)
    n1 = n // 2
    n2 = n - n1
    lo, hi = row_partition(n2, world, B)[rank]
    a11 = a[:n1, :n1].contiguous() if rank == 0 else None
    a21 = a[:n1, n1 + lo:n1 + hi].contiguous()      # rows n1+lo.., cols 0..n1
    a22 = a[n1:, n1 + lo:n1 + hi].contiguous()      # rows n1+lo.., cols n1..
    return a, a11, a21, a22


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
    a, a11, a21, a22 = _pieces(tc, N, SEED, 1, 0)
    res = potrf_top_split(N, B, CFG, a11=a11, a21_rows=a21, a22_rows=a22)
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


def _rank_main(rank, world, port, outdir):
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
    _, a11, a21, a22 = _pieces(tc, N, SEED, world, rank)
    res = potrf_top_split(N, B, CFG, a11=a11, a21_rows=a21, a22_rows=a22)
    np.save(os.path.join(outdir, f"l21_{rank}.npy"), res.l21_rows.cpu().numpy())
    if rank == 0:
        np.save(os.path.join(outdir, "l11.npy"), res.l11.cpu().numpy())
        np.save(os.path.join(outdir, "l22.npy"), res.l22.cpu().numpy())
    with open(os.path.join(outdir, f"status_{rank}"), "w") as f:
        f.write(res.status)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_distributed_two_ranks_one_gpu_bit_identical(tc, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    for r in range(2):
        assert open(tmp_path / f"status_{r}").read() == "ok"
    ref = _single(tc, N, SEED).cpu().numpy()
    n1 = N // 2
    parts = row_partition(N - n1, 2, B)
    assert np.array_equal(np.tril(np.load(tmp_path / "l11.npy").T), np.tril(ref[:n1, :n1].T))
    for r, (lo, hi) in enumerate(parts):
        assert np.array_equal(np.load(tmp_path / f"l21_{r}.npy"), ref[:n1, n1 + lo:n1 + hi])
    assert np.array_equal(np.tril(np.load(tmp_path / "l22.npy").T), np.tril(ref[n1:, n1:].T))
