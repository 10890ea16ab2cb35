"""Distributed single factorization across GPUs (BASELINE config C5;
SURVEY 8(e)): the top split of an order-N tree_potrf (tree.cpp:106-125) with
its TRSM and SYRK split by rows over the ranks.

    n1 = N/2, n2 = N - n1;  A = [[A11, .], [A21, A22]],  p = the panel level
    1. rank 0:   L11 = tree_potrf(A11)                  (a whole-plan factorization)
    2. rank 0 forms rn_p(L11) -- all tree_trsm ever reads of L (kernels.cpp:29,
       78) -- as a row-major level image and broadcasts it (NCCL over NVLink;
       FP16 at C5: n1^2 * 2 bytes) straight into every rank's TRSM workspace
    3. all-reduce(max) of max|A21| -- the panel's alpha is one scalar over the
       whole block (tree.cpp:81-88), so every rank quantizes with the same one
    4. rank r:   its TRSM rows of A21 <- tree_trsm(quantize(A21_r), L11),
                 dequantize (TRSM rows are independent, tree.cpp:133-134)
    5. every rank broadcasts its solved rows' level image (exact: the stored
       values are level-rounded) into every rank's SYRK workspace
    6. rank r:   tree_syrk(A22, A21) on A22's SYRK rows R_r (GEMM output rows
                 are independent); R_r balance the lower-triangle work
    7. A22's rows go to rank 0 (point to point);  rank 0: L22 = tree_potrf(A22)

Every block gets the same operations in the same order as on one device, so
the distributed factor is bit-identical to the single-device one
(tests/test_distributed.py checks it with 1, 2 and 4 ranks).

Memory (the pieces are compact plans, Plan.panel_trsm_ext /
panel_syrk_rows_ext: no square operand copies, level buffers only for the
rows a rank touches): at N = 131072 on 8 GPUs rank 0 peaks near 143 GB
(A11/L11 and A22/L22 in doubles 34.4 GB each, the order-65536 plan 25.8 GB,
its pieces ~50 GB), the others near 30 GB (memory_plan, tested against the
180 GB of a B200 with a 150 GB budget).  Not measured on hardware: the
driver's boxes have one GPU.  The A11 and A22 factorizations stay serial on
rank 0 (the split is one level deep).

Collectives run on NCCL; with a gloo group (tests: ranks sharing one GPU)
they are staged through host memory.  Device tensors use the package's
column-major layout (``to_device``: t[j, i] = A(i, j)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


def row_partition(n2: int, world: int, align: int) -> list:
    """contiguous row ranges of [0, n2) per rank, bounds multiples of `align`,
    equal row counts (the TRSM split: rows cost the same)"""
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


def leaf_starts(n: int, b: int, r0: int = 0) -> list:
    """first rows of the diagonal leaves of an order-n tree (build_node,
    tree.cpp:42-66: n1 = floor(n/2), leaf iff n <= b), plus n"""
    out = []

    def rec(r, m):
        if m <= b:
            out.append(r)
            return
        h = m // 2
        rec(r, h)
        rec(r + h, m - h)
    rec(r0, n)
    return out + [r0 + n]


def syrk_partition(n2: int, b: int, world: int) -> list:
    """row ranges of A22 per rank for the SYRK: the work of rows [lo, hi) of
    a lower-triangular update grows like hi^2 - lo^2, so the bounds sit near
    n2 sqrt(r / world), moved to the nearest diagonal-leaf boundary (a leaf
    may not straddle two ranks)"""
    if world < 1:
        raise ValueError("bad partition arguments")
    cuts = leaf_starts(n2, b)
    out, lo = [], 0
    for r in range(1, world + 1):
        if r == world:
            hi = n2
        else:
            target = n2 * math.sqrt(r / world)
            hi = min((c for c in cuts if c >= lo), key=lambda c: abs(c - target))
        out.append((lo, hi))
        lo = hi
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
    l21_rows: object = None  # every rank: its solved TRSM rows of A21 (n1 x m_r tensor)
    l22: object = None      # rank 0: factored A22
    rows: tuple = (0, 0)    # this rank's TRSM rows of A21
    syrk_rows: tuple = (0, 0)  # this rank's SYRK rows of A22
    status: str = "ok"      # the first failure in the reference's order, on every rank
    detail: str = ""
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
            if self.rank != src:
                t.copy_(h)
        else:
            self.dist.broadcast(t, src, group=self.group)
        return t

    def _scalar(self, x: float, op) -> float:
        import torch
        if not self.on or self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.host else "cuda")
        self.dist.all_reduce(t, op=op, group=self.group)
        return float(t.item())

    def allreduce_max(self, x: float) -> float:
        return self._scalar(x, self.dist.ReduceOp.MAX) if self.on else x

    def allreduce_min(self, x: float) -> float:
        return self._scalar(x, self.dist.ReduceOp.MIN) if self.on else x

    def send(self, t, dst):
        self.dist.send(t.cpu() if self.host else t, dst, group=self.group)

    def recv(self, t, src):
        if self.host:
            h = t.cpu()
            self.dist.recv(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.recv(t, src, group=self.group)

    def gather_object(self, obj):
        if not self.on or self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        if self.on and self.world > 1:
            self.dist.barrier(group=self.group)


_STEP_NAMES = {1: "A11", 4: "panel TRSM", 6: "panel SYRK", 8: "A22"}


def potrf_top_split(n: int, b: int, config, a11=None, a21_rows=None, a22_rows=None, l22=None, group=None,
                    cache: dict | None = None) -> DistResult:
    """Distributed tree_potrf of an order-n matrix (quantization on).

    Inputs (device float64, column-major):
      rank 0:     ``a11`` (n1 x n1, factored in place) and ``l22`` (n2 x n2:
                  receives A22's updated lower part and is factored in place);
      every rank: ``a21_rows`` = A21[T_r, :] (tensor (n1, m_r)) with
                  T_r = row_partition(n2, world, b)[rank], overwritten by its
                  solved rows, and ``a22_rows`` = A22[S_r, :] (tensor
                  (n2, s_r)) with S_r = syrk_partition(n2, b, world)[rank],
                  overwritten by its updated rows.
    ``cache`` (a dict kept by the caller) keeps the plans -- their device
    workspace and CUDA graphs -- across calls.  The status is the first
    failure in the reference's order (steps, then ranks = rows), the same on
    every rank; later steps are skipped once one failed.
    """
    import torch
    import paper_2601_08082_b200 as tc

    cfg = tc._cfg(config)
    levels = cfg.levels
    co = _Coll(group)
    n1 = n // 2
    n2 = n - n1
    tparts = row_partition(n2, co.world, b)
    sparts = syrk_partition(n2, b, co.world)
    lo_t, hi_t = tparts[co.rank]
    lo_s, hi_s = sparts[co.rank]
    m_t = hi_t - lo_t
    res = DistResult(rows=(lo_t, hi_t), syrk_rows=(lo_s, hi_s))
    sub = shifted_levels(levels)
    p = levels[0]
    cache = {} if cache is None else cache

    def plan(key, make):
        if key not in cache:
            cache[key] = make()
        return cache[key]

    fail = [None]  # (step, rank, status, detail) of this rank's first failure

    def note(step, st):
        if st.status != "ok" and fail[0] is None:
            fail[0] = (step, co.rank, st.status, st.detail)

    def agree() -> bool:
        """every rank learns the earliest failure so far; True if none"""
        key = float(fail[0][0] * co.world + fail[0][1]) if fail[0] else math.inf
        first = co.allreduce_min(key)
        if math.isinf(first):
            return True
        step, owner = divmod(int(first), co.world)
        infos = co.gather_object(fail[0])
        _, _, res.status, res.detail = infos[owner]
        return False

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    co.barrier()
    torch.cuda.synchronize()
    ev0.record()

    # 1. factor A11 on rank 0 (the big tree's diag1: levels shifted by one)
    whole = lambda: tc.Plan(n1, b, sub)  # noqa: E731
    if co.rank == 0:
        note(1, plan("p11", whole).factor_device(a11))
        res.l11 = a11
    if not agree():
        return _done(res, ev0, ev1)

    # 2. rn_p(L11) from rank 0 straight into every rank's TRSM workspace
    ldw = (n1 + 63) // 64 * 64  # row stride of the pieces' level buffers (Plan::ldw)
    pt = plan("pt", lambda: tc.Plan.panel_trsm_ext(n1, m_t, b, cfg)) if m_t > 0 else None
    if pt is not None:
        tbuf, t_lo = pt.level_buffer(p)   # rows [0, n1 + m_t)
        assert t_lo == 0 and tbuf.shape[1] == ldw
    else:
        tbuf, t_lo = torch.empty((n1, ldw), dtype=exact_dtype(p), device="cuda"), 0
    l11_img = tbuf[:n1]
    if co.rank == 0:
        tc.level_image_device(a11, n1, n1, p, l11_img, l11_img.shape[1], lower=True)
    co.broadcast(l11_img, 0)

    # 3. global max |A21| (the panel alpha)
    amax = tc.absmax_device(a21_rows, m_t, n1) if m_t > 0 else 0.0
    amax = co.allreduce_max(amax)

    # 4. solve this rank's rows of A21 against L11
    if pt is not None:
        pt.set_external_absmax(amax)
        note(4, pt.factor_device(a21_rows))
    res.l21_rows = a21_rows
    if not agree():
        return _done(res, ev0, ev1)

    # 5. every rank's solved rows (level image) into every SYRK workspace,
    #    at panel rows [hi_s + lo_r, hi_s + hi_r)
    ps = plan("ps", lambda: tc.Plan.panel_syrk_rows_ext(n2, n1, b, cfg, lo_s, hi_s)) if hi_s > lo_s else None
    if ps is not None:
        sbuf, s_lo = ps.level_buffer(p)
        same = sbuf.shape[1] == ldw  # the same row stride: receive in place
    for r, (lo, hi) in enumerate(tparts):
        if hi <= lo:
            continue
        dst = sbuf[hi_s + lo - s_lo:hi_s + hi - s_lo] if ps is not None else None
        if co.rank == r:
            piece = tbuf[n1:n1 + (hi - lo)]  # full rows: contiguous
        elif dst is not None and same:
            piece = dst
        else:
            piece = torch.empty((hi - lo, ldw), dtype=tbuf.dtype, device="cuda")
        co.broadcast(piece, r)
        if dst is not None and dst.data_ptr() != piece.data_ptr():
            dst[:, :n1].copy_(piece[:, :n1])

    # 6. this rank's rows of A22 <- A22 - A21 A21^T (tree_syrk)
    if ps is not None:
        note(6, ps.factor_device(a22_rows))
    if not agree():
        return _done(res, ev0, ev1)

    # 7. A22's rows to rank 0, then factor A22 there
    if co.rank == 0:
        for r, (lo, hi) in enumerate(sparts):
            if hi <= lo:
                continue
            if r == 0:
                l22[:, lo:hi].copy_(a22_rows)
            else:
                tmp = torch.empty((n2, hi - lo), dtype=torch.float64, device="cuda")
                co.recv(tmp, r)
                l22[:, lo:hi].copy_(tmp)
                del tmp
        p22 = plan("p11", whole) if n2 == n1 else plan("p22", lambda: tc.Plan(n2, b, sub))
        note(8, p22.factor_device(l22))
        res.l22 = l22
    elif hi_s > lo_s:
        co.send(a22_rows.contiguous(), 0)
    agree()
    return _done(res, ev0, ev1)


def _done(res, ev0, ev1):
    import torch
    ev1.record()
    torch.cuda.synchronize()
    res.device_ms = ev0.elapsed_time(ev1)
    return res


def memory_plan(n: int, b: int, config, world: int) -> list:
    """device bytes each rank holds at its peak in potrf_top_split (plans'
    workspaces from the planner -- no device needed -- plus the caller's
    operands and the transient receive buffers), for the memory budget of
    BASELINE config C5 (tests/test_distributed.py)"""
    import paper_2601_08082_b200 as tc
    cfg = tc._cfg(config)
    n1, n2 = n // 2, n - n // 2
    tparts, sparts = row_partition(n2, world, b), syrk_partition(n2, b, world)
    whole = tc.Plan(n1, b, shifted_levels(cfg.levels)).device_bytes()
    esz = (2, 4, 8)[cfg.levels[0]]
    out = []
    for r in range(world):
        m_t = tparts[r][1] - tparts[r][0]
        s_r = sparts[r][1] - sparts[r][0]
        pt = tc.Plan.panel_trsm_ext(n1, max(m_t, 1), b, cfg).device_bytes()
        ps = tc.Plan.panel_syrk_rows_ext(n2, n1, b, cfg, *sparts[r]).device_bytes() if s_r > 0 else 0
        mine = pt + ps + 8 * (m_t * n1 + s_r * n2)          # pieces + this rank's A21 / A22 rows
        mine += esz * max(h - l for l, h in tparts) * n1      # a received panel piece (worst case)
        if r == 0:
            mine += 8 * (n1 * n1 + n2 * n2) + whole           # A11/L11, A22/L22, the order-n1 plan
            mine += 8 * n2 * max((h - l for l, h in sparts[1:]), default=0)  # one A22 piece in flight
        out.append(mine)
    return out


def synthetic_pieces(n: int, b: int, seed: int, world: int, rank: int):
    """this rank's inputs of a device-generated SPD matrix of spd_generate's
    distribution (off-diagonal uniform [0, 1), n on the diagonal; only the
    lower triangle is read): (a11 on rank 0 else None, a21 TRSM rows,
    a22 SYRK rows, l22 buffer on rank 0 else None)"""
    import torch
    n1, n2 = n // 2, n - n // 2
    lo, hi = row_partition(n2, world, b)[rank]
    slo, shi = syrk_partition(n2, b, world)[rank]
    g = torch.Generator(device="cuda").manual_seed(int(seed) * 1000 + rank)
    a11 = l22 = None
    if rank == 0:
        r = torch.rand((n1, n1), dtype=torch.float64, device="cuda", generator=g)
        a11 = (r + r.T).mul_(0.5)
        a11.diagonal().add_(float(n))
        del r
        l22 = torch.empty((n2, n2), dtype=torch.float64, device="cuda")
    a21 = torch.rand((n1, hi - lo), dtype=torch.float64, device="cuda", generator=g)
    a22 = torch.rand((n2, shi - slo), dtype=torch.float64, device="cuda", generator=g)
    idx = torch.arange(shi - slo, device="cuda")
    a22[slo + idx, idx] += float(n)
    return a11, a21, a22, l22
