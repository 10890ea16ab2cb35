"""Distributed single factorization across GPUs (BASELINE config C5;
SURVEY 8(e)): the top split of an order-N tree_potrf (tree.cpp:106-125) with
its TRSM and SYRK split by rows over the ranks.

    n1 = N/2, n2 = N - n1;  A = [[A11, .], [A21, A22]]
    1. rank 0:   L11 = tree_potrf(A11)                  (a whole-plan factorization)
    2. broadcast L11 (NCCL over NVLink; the lowest exact float format)
    3. all-reduce(max) of max|A21| -- the panel's alpha is one scalar over the
       whole block (tree.cpp:81-88), so every rank quantizes with the same one
    4. rank r:   its rows of A21 <- tree_trsm(quantize(A21_r), L11), dequantize
                 (Plan.panel_trsm; TRSM rows are independent, tree.cpp:133-134)
    5. all-gather the solved A21 (its level's exact format, FP16 at C5)
    6. rank r:   tree_syrk(A22, A21) on A22's rows R_r (Plan.panel_syrk_rows;
                 GEMM output rows are independent)
    7. gather A22's rows to rank 0;  rank 0: L22 = tree_potrf(A22)

Every block gets the same operations in the same order as on one device, so
the distributed factor is bit-identical to the single-device one
(tests/test_distributed.py checks it).  Device tensors use the package's
column-major layout (``to_device``: t[j, i] = A(i, j)).

Collectives run on NCCL; with a gloo group (tests: two ranks sharing one GPU)
they are staged through host memory.
"""
from __future__ import annotations

from dataclasses import dataclass


def row_partition(n2: int, world: int, align: int) -> list:
    """contiguous row ranges of [0, n2) per rank, bounds multiples of `align`
    (the leaf size: a diagonal leaf never straddles two ranks)"""
    if world < 1 or align < 1:
        raise ValueError("bad partition arguments")
    units = (n2 + align - 1) // align
    base, extra = divmod(units, world)
    out, u = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        lo, hi = min(n2, u * align), min(n2, (u + k) * align)
        out.append((lo, hi))
        u += k
    return out


def shifted_levels(levels) -> tuple:
    """the levels of a depth-1 subtree as a standalone tree: at_depth(1 + d)"""
    lv = tuple(levels)
    return lv[1:] if len(lv) > 1 else lv


def exact_dtype(max_level: int):
    import torch
    return {0: torch.float16, 1: torch.float32}.get(max_level, torch.float64)


@dataclass
class DistResult:
    l11: object = None      # rank 0: factored A11 (device, column-major)
    l21_rows: object = None  # every rank: its solved rows of A21 (n1 x m_r tensor view)
    l22: object = None      # rank 0: factored A22
    rows: tuple = (0, 0)    # this rank's rows of A21 / A22
    status: str = "ok"
    device_ms: float = 0.0  # this rank's device time of steps 1-7


class _Coll:
    """collectives on device tensors; staged through the host on gloo"""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.host = self.on and dist.get_backend(group) == "gloo"

    def broadcast(self, t, src=0):
        if not self.on or self.world == 1:
            return t
        if self.host:
            h = t.cpu()
            self.dist.broadcast(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src, group=self.group)
        return t

    def allreduce_max(self, x: float) -> float:
        import torch
        if not self.on or self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.host else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allgather(self, t, sizes):
        """all ranks' tensors (shape (C, sizes[r])) -> list in rank order"""
        import torch
        if not self.on or self.world == 1:
            return [t]
        dev = torch.device("cpu") if self.host else t.device
        outs = [torch.empty((t.shape[0], s), dtype=t.dtype, device=dev) for s in sizes]
        src = t.cpu() if self.host else t
        self.dist.all_gather(outs, src.contiguous(), group=self.group)
        return [o.to(t.device) for o in outs]

    def barrier(self):
        if self.on and self.world > 1:
            self.dist.barrier(group=self.group)


def potrf_top_split(n: int, b: int, config, a11=None, a21_rows=None, a22_rows=None, group=None,
                    cache: dict | None = None) -> DistResult:
    """Distributed tree_potrf of an order-n matrix (quantization on).

    Inputs (device float64, column-major): rank 0 passes ``a11`` (n1 x n1,
    factored in place); every rank passes ``a21_rows`` = A21[R_r, :]
    (tensor (n1, m_r)) and ``a22_rows`` = A22[R_r, :] (tensor (n2, m_r)),
    with R_r = row_partition(n2, world, b)[rank].  Returns the factor pieces.
    ``cache`` (a dict kept by the caller) keeps the plans -- their device
    workspace and CUDA graphs -- across calls.
    """
    import torch
    import paper_2601_08082_b200 as tc

    cfg = tc._cfg(config)
    levels = cfg.levels
    co = _Coll(group)
    n1 = n // 2
    n2 = n - n1
    parts = row_partition(n2, co.world, b)
    lo, hi = parts[co.rank]
    m = hi - lo
    res = DistResult(rows=(lo, hi))
    sub = shifted_levels(levels)
    cache = {} if cache is None else cache

    def plan(key, make):
        if key not in cache:
            cache[key] = make()
        return cache[key]

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    co.barrier()
    torch.cuda.synchronize()
    ev0.record()

    # 1-2. factor A11 on rank 0, broadcast L11 in the lowest exact format
    l11_t = exact_dtype(max(sub))
    if co.rank == 0:
        p11 = plan("p11", lambda: tc.Plan(n1, b, sub))
        st = p11.factor_device(a11)
        if st.status != "ok":
            res.status = st.status
        l11_x = a11.to(l11_t)
        res.l11 = a11
    else:
        l11_x = torch.empty((n1, n1), dtype=l11_t, device="cuda")
    co.broadcast(l11_x, 0)

    # 3. global max |A21| (the panel alpha)
    amax = tc.absmax_device(a21_rows, m, n1) if m > 0 else 0.0
    amax = co.allreduce_max(amax)

    # 4. solve this rank's rows of A21 against L11
    p = levels[0]
    if m > 0:
        t = torch.empty((n1, n1 + m), dtype=torch.float64, device="cuda")
        t[:, :n1].copy_(l11_x)
        t[:, n1:].copy_(a21_rows)
        del l11_x
        pt = plan("pt", lambda: tc.Plan.panel_trsm(n1, m, b, cfg))
        pt.set_external_absmax(amax)
        st = pt.factor_device(t)
        if st.status != "ok":
            res.status = st.status
        x_r = t[:, n1:]
    else:
        x_r = torch.empty((n1, 0), dtype=torch.float64, device="cuda")

    # 5. all-gather the solved panel (exact in its level's format)
    xt = exact_dtype(p)
    pieces = co.allgather(x_r.to(xt), [h - l for (l, h) in parts])
    res.l21_rows = x_r

    # 6. this rank's rows of A22 <- A22 - A21 A21^T (tree_syrk)
    s = torch.zeros((n2, 2 * n2), dtype=torch.float64, device="cuda")
    for (l2, h2), piece in zip(parts, pieces):
        if h2 > l2:
            s[:n1, n2 + l2:n2 + h2].copy_(piece)
    del pieces
    if m > 0:
        s[:, lo:hi].copy_(a22_rows)
        ps = plan("ps", lambda: tc.Plan.panel_syrk_rows(n2, n1, b, cfg, lo, hi))
        st = ps.factor_device(s)
        if st.status != "ok":
            res.status = st.status
    # 7. A22 to rank 0 (exact in the widest level of the A22 tree), factor it
    a22t = exact_dtype(max(sub))
    mine = s[:n2, lo:hi].to(a22t)
    del s
    got = co.allgather(mine, [h - l for (l, h) in parts])
    if co.rank == 0:
        a22 = torch.empty((n2, n2), dtype=torch.float64, device="cuda")
        for (l2, h2), piece in zip(parts, got):
            if h2 > l2:
                a22[:, l2:h2].copy_(piece)
        p22 = plan("p22", lambda: tc.Plan(n2, b, sub))
        st = p22.factor_device(a22)
        if st.status != "ok":
            res.status = st.status
        res.l22 = a22
    del got
    ev1.record()
    torch.cuda.synchronize()
    res.device_ms = ev0.elapsed_time(ev1)
    return res


def synthetic_pieces(n: int, b: int, seed: int, world: int, rank: int):
    """this rank's inputs of a device-generated SPD matrix of spd_generate's
    distribution (off-diagonal uniform [0, 1), n on the diagonal; only the
    lower triangle is read): (a11 on rank 0 else None, a21_rows, a22_rows)"""
    import torch
    n1, n2 = n // 2, n - n // 2
    lo, hi = row_partition(n2, world, b)[rank]
    g = torch.Generator(device="cuda").manual_seed(int(seed) * 1000 + rank)
    a11 = None
    if rank == 0:
        r = torch.rand((n1, n1), dtype=torch.float64, device="cuda", generator=g)
        a11 = (r + r.T).mul_(0.5)
        a11.diagonal().add_(float(n))
    a21 = torch.rand((n1, hi - lo), dtype=torch.float64, device="cuda", generator=g)
    a22 = torch.rand((n2, hi - lo), dtype=torch.float64, device="cuda", generator=g)
    idx = torch.arange(hi - lo, device="cuda")
    a22[lo + idx, idx] += float(n)
    return a11, a21, a22
