"""Batched POTRF + POTRS (BASELINE config C4) and its multi-GPU sharding.

CPU: the shard partition and the cross-rank reduction on a world_size-2
gloo group (the N>1 host path; there is no data-path collective to test).
GPU: a batch through tc_batch_run against the oracle (status, backward
error, solve residual), including a failing system in the middle of a batch.
"""
import os
import socket

import numpy as np
import pytest

from paper_2601_08082_b200.batch import ShardResult, reduce_results, shard


def test_shard_partition_properties():
    for count in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            parts = [list(shard(count, world, r)) for r in range(world)]
            flat = [k for p in parts for k in p]
            assert flat == list(range(count))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(64, world, rank)
    local = ShardResult(len(mine), rank, 10.0 + rank, 1e-15 * (rank + 1))
    tot = reduce_results(local)
    q.put((rank, list(mine)[:1], tot.systems, tot.failed, tot.device_ms, tot.worst_residual))
    dist.destroy_process_group()


def test_sharded_reduction_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out[0][1] == [0] and out[1][1] == [32]
    for _, _, systems, failed, ms, res in out:
        assert systems == 64 and failed == 1 and ms == 11.0 and res == pytest.approx(2e-15)


@pytest.mark.gpu
def test_batch_matches_oracle(tc, oracle):
    import torch
    from pyoracle import parse_levels
    n, b, cfg = 512, 64, "[F16, F16, F32]"
    seeds = [3, 4, 5, 6, 7]
    mats = [oracle.spd_generate(n, s) for s in seeds]
    mats[2] = mats[2].copy(order="F")
    mats[2][100, 100] = -1.0  # indefinite: NotPositiveDefinite at row 100 (oracle decides)
    a_dev = [tc.to_device(m) for m in mats]
    a0 = [x.clone() for x in a_dev]
    rhs = [torch.from_numpy(m.sum(axis=1)).reshape(1, n).to("cuda") for m in mats]
    rhs0 = [x.clone() for x in rhs]
    batch = tc.Batch(n, b, cfg, True, concurrency=2)
    st = batch.run(a_dev, rhs)
    for k, m in enumerate(mats):
        st_o, det_o, _, rel_o, _ = oracle.factor(m, b, parse_levels(cfg))
        assert st[k] == st_o, (k, st[k], st_o, det_o)
        if st_o == "ok":
            rel = tc.factorization_error_device(a0[k], a_dev[k])
            assert rel <= 2 * rel_o, (k, rel, rel_o)
            res = tc.solve_residual_device(a0[k], rhs[k][0].contiguous(), rhs0[k][0].contiguous())
            assert res < 1e-5, (k, res)


@pytest.mark.gpu
def test_batch_rank_driver_single_gpu(tc):
    from paper_2601_08082_b200.batch import run_batch_on_rank
    local, tot, flops = run_batch_on_rank(4, 1024, 128, "[F16, F16, F16, F32]", seed0=11, concurrency=2,
                                          in_flight=4)
    assert local.systems == 4 and tot.failed == 0
    assert tot.worst_residual < 1e-5 and flops > 0 and tot.device_ms > 0


@pytest.mark.gpu
def test_batch_solve_orders_agree(tc, oracle):
    """solve_order 0 (every factorization, then all solves in one batched
    launch sequence) and 1 (each solve behind its factorization, single-system
    launches) give bit-identical factors and solutions, with 2 RHS, more
    systems than plans, and one system without right-hand sides"""
    import torch
    n, b, cfg = 768, 64, "[F16, F16, F32]"
    mats = [oracle.spd_generate(n, s) for s in range(5)]
    out = []
    for order in (0, 1):
        a_dev = [tc.to_device(m) for m in mats]
        rhs = [torch.from_numpy(np.stack([m.sum(axis=1), m[:, 0]])).to("cuda").contiguous() for m in mats]
        rhs[3] = None
        batch = tc.Batch(n, b, cfg, True, concurrency=2)
        batch.set_option("solve_order", order)
        st = batch.run(a_dev, rhs)
        assert all(s == "ok" for s in st)
        out.append(([x.cpu().numpy() for x in a_dev], [None if x is None else x.cpu().numpy() for x in rhs]))
    for k in range(len(mats)):
        assert np.array_equal(np.tril(out[0][0][k].T), np.tril(out[1][0][k].T))
        if k != 3:
            assert np.array_equal(out[0][1][k], out[1][1][k])


@pytest.mark.gpu
def test_c4_unit_matches_golden(tc):
    """BASELINE config C4's unit system at full size (N=16384, b=256,
    [F16, F16, F16, F32], spd_generate seeds 0 and 1 -- bit-identical device
    generation) through tc_batch_run: status and flops exactly, backward
    error and the solve residual for b = A * ones within 2x of the oracle's
    (tests/golden/c4.json, made by tests/golden/make_golden_c4.py)"""
    import json
    import torch
    with open(os.path.join(os.path.dirname(__file__), "golden", "c4.json")) as f:
        gold = json.load(f)
    n, b, cfg = gold["n"], gold["b"], gold["config"]
    assert tuple(tc.flop_breakdown(n, b, cfg).as_tuple()) == tuple(gold["cases"][0]["flops"])
    batch = tc.Batch(n, b, cfg, True, concurrency=2)
    a_list, keep, rhs, rhs0 = [], [], [], []
    for case in gold["cases"]:
        a = tc.spd_generate_device(n, case["seed"])
        bv = a.cpu().numpy().T.sum(axis=1)  # b = A * ones exactly as the golden script sums it
        a_list.append(a)
        keep.append(a.clone())
        rhs.append(torch.from_numpy(bv).reshape(1, n).to("cuda"))
        rhs0.append(rhs[-1].clone())
    st = batch.run(a_list, rhs)
    for k, case in enumerate(gold["cases"]):
        assert st[k] == case["status"] == "ok"
        rel = tc.factorization_error_device(keep[k], a_list[k])
        res = tc.solve_residual_device(keep[k], rhs[k][0].contiguous(), rhs0[k][0].contiguous())
        assert rel <= 2 * case["rel_error"], (case["seed"], rel, case["rel_error"])
        assert res <= 2 * case["potrs_residual"], (case["seed"], res, case["potrs_residual"])
