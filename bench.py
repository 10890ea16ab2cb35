#!/usr/bin/env python3
"""bench.py -- mixed-precision POTRF TFLOP/s at N=65536 on B200 (BASELINE.json).

Workload (BASELINE config C3): A = spd_generate(65536, 42)
(analysis.cpp:12-28, bit-identical, generated on the device), leaf b = 256,
precision tree "[F16, F16, F16, F32]", quantization on.  One step = one full
tree_potrf of the device-resident matrix (import .. export, i.e. caller
doubles in, caller doubles out).  Metric = n(n+1)(2n+1)/6 flops per step
(analysis.cpp:66-68) / device time.  Inputs (34 GB) exceed L2, so no flush.

Multi-GPU (torchrun): the path shards as independent systems (SURVEY 8e, C4
style): every rank factors its own N=65536 matrix, no data-path collective;
`value` = all ranks' flops / max-over-ranks time ("scaling": "weak").

--impl reference: the reference's own CPU implementation (oracle/_ref, the
compiled /root/reference sources) timed on the host cores, every core running
one factor_matrix of a bounded sample (N=1536, same b and tree) per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = "[F16, F16, F16, F32]"
N_DEFAULT, B_DEFAULT, SEED = 65536, 256, 42
METRIC = "mixed-precision POTRF TFLOP/s at N=65536 (1 B200) + rel. backward error"


def potrf_flops(n: int) -> int:
    return n * (n + 1) * (2 * n + 1) // 6


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region"""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if x > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------- reference
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from multiprocessing import Pool

    from pyoracle import Reference
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    cores = os.cpu_count() or 1
    ns = args.ref_n
    total = args.warmup + args.steps
    times = []
    with Pool(cores) as pool:
        for step in range(total):
            t0 = time.perf_counter()
            pool.map(_ref_worker, [(ns, args.b, SEED + k) for k in range(cores)])
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                times.append(dt)
    per_step = statistics.mean(times)
    tflops = cores * potrf_flops(ns) / per_step / 1e12
    sample = (f"{cores} concurrent factor_matrix(spd_generate({ns}, seed), b={args.b}, {CFG}) per step, "
              f"one per host core (reference is single-threaded); N={args.n} itself is infeasible on CPU")
    line = {"metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64-emulated(F16/F32 rounding)", "data": "synthetic spd_generate",
            "impl": "reference",
            "config": {"workload": f"C3 sample: N={ns} b={args.b} {CFG} (host CPU)", "n": ns, "b": args.b,
                       "precision_tree": CFG},
            "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _ref_worker(arg):
    ns, b, seed = arg
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference, parse_levels
    r = Reference()
    a = r.spd_generate(ns, seed)
    return r.time_factor_ms(a, b, parse_levels(CFG), True)


def cpu_baseline_sample(args):
    """the compiled reference on one host core, bounded sample (rank 0, N=1)"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, Reference, parse_levels
    ns = args.cpu_n
    if Reference.available():
        r = Reference()
        a = r.spd_generate(ns, SEED)
        ms = r.time_factor_ms(a, args.b, parse_levels(CFG), True)
        kind = "reference"
    else:
        o = Oracle()
        o.set_threads(1)
        a = o.spd_generate(ns, SEED)
        t0 = time.perf_counter()
        o.factor(a, args.b, parse_levels(CFG))
        ms = (time.perf_counter() - t0) * 1e3
        kind = "port"
    return {"value": potrf_flops(ns) / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": kind,
            "sample": f"one factor_matrix(spd_generate({ns}, {SEED}), b={args.b}, {CFG}) on 1 host core: "
                      f"{ms / 1e3:.1f} s (N={args.n} is weeks of CPU time)"}


# --------------------------------------------------------------------- ours
def allreduce_max(x: float, host: bool) -> float:
    """max over ranks of a host float (device tensor on NCCL, CPU on gloo)"""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if host else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2601_08082_b200 as tc

    ws, rank, local = dist_env()
    ndev = torch.cuda.device_count()
    # one process per GPU; with fewer GPUs than ranks (a dry run of --gpus N
    # on a smaller box) ranks share devices and the host-side reductions go
    # over gloo (NCCL refuses two ranks on one device)
    shared = ws > ndev
    torch.cuda.set_device(local % ndev)
    if ws > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, b = args.n, args.b
    peaks, peak_kind = measured_peaks()

    # inputs: spd_generate(n, seed + rank) straight into HBM (column-major)
    a = tc.spd_generate_device(n, SEED + rank)
    l = torch.empty_like(a)
    plan = tc.Plan(n, b, CFG, True)
    st = plan.factor_device(a, l)  # builds + captures the CUDA graph
    if st.status != "ok":
        raise SystemExit(f"factorization failed: {st.status} {st.detail}")
    stats = plan.stats()
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.factor_device(a, l, stream=stream, sync=False)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            plan.factor_device(a, l, stream=stream, sync=False)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    st = plan.status()
    if ws > 1:
        ms = allreduce_max(ms, shared)
    flops = potrf_flops(n)
    value = ws * args.steps * flops / (ms * 1e-3) / 1e12
    ms_per_step = ms / args.steps

    # accuracy of the timed factorization (device FP64 metric, analysis.cpp:30-62)
    rel = tc.factorization_error_device(a, l) if st.status == "ok" else float("nan")

    # roofline of the dominant kernel: tcgen05 FP16 GEMM, per-op device time
    # from a serialized profiling replay (kernel timed alone -> burst peak)
    op_ms = plan.profile(a, l, stream=stream)
    tc_ms, tc_fl, tot_ms = 0.0, 0.0, sum(op_ms)
    # per-launch roofline of the same kernel: each launch is bound by the
    # slower of its flops at the tensor peak and its algorithmic bytes (A, B
    # read once, C written -- and read when beta != 0) at the HBM peak; the
    # small-K trailing updates are HBM-bound on their C traffic
    t_bound, n_hbm, alg_bytes = 0.0, 0, 0.0
    by_type = {}
    for i, t in enumerate(op_ms):
        info = plan.op_info(i)
        key = info["type"] + ("/" + info["gclass"] if info["gclass"] else "")
        e = by_type.setdefault(key, [0.0, 0.0, 0])
        e[0] += t
        e[1] += info["flops"]
        e[2] += 1
        if info["gclass"] == "tc16":
            tc_ms += t
            tc_fl += info["flops"]
            nbytes = 0.0
            for pr in plan.op_probs(i):
                beta = 0 if pr["a_kwrap"] else 1  # in-place inverse solves write C only
                celems = pr["m"] * pr["n"] / (2.0 if pr["lower"] else 1.0)
                nbytes += 2.0 * pr["m"] * (pr["a_kwrap"] or pr["k"]) + 2.0 * pr["n"] * pr["k"]
                nbytes += celems * (2.0 if pr["exec_level"] == 0 else 4.0) * (1 + beta)
            alg_bytes += nbytes
            tb_t = info["flops"] / (peaks["bf16_tflops"] * 1e12) * 1e3
            tb_h = nbytes / (peaks["hbm_gbs"] * 1e9) * 1e3
            t_bound += max(tb_t, tb_h)
            n_hbm += tb_h > tb_t
    achieved = tc_fl / (tc_ms * 1e-3) / 1e12 if tc_ms else 0.0
    # DRAM traffic per launch of the same kernel, from the committed ncu
    # launch list of this command (profiles/ncu_traffic.json)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {"bound": "tensor",
                "kernel": "k_gemm_tc / k_gemm_tc2 (tcgen05 kind::f16, FP32 accumulate; CTA pairs for >= 512 tiles)",
                "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16_tflops"], "traffic": traffic, "traffic_unit": "bytes/launch (ncu)",
                "peak_kind": f"{peak_kind} bf16 burst (MEASURED_PEAKS.json)",
                "share_of_step": tc_ms / tot_ms if tot_ms else None,
                "launches": by_type.get("gemm/tc16", [0, 0, 0])[2],
                # A, B read once, C written (and read when beta != 0): what the
                # ncu `traffic` figure is compared against
                "algorithmic_bytes_per_launch": alg_bytes / max(1, by_type.get("gemm/tc16", [0, 0, 0])[2]),
                "per_launch_bound": {"frac": t_bound / tc_ms if tc_ms else None, "hbm_bound_launches": n_hbm,
                                     "note": "sum over launches of max(flops / tensor peak, algorithmic bytes / "
                                             "HBM peak) / sum of measured launch times"}}
    del op_ms

    # e2e: the public host entry point (tc_potrf_host, reference TileView
    # contract): pinned host doubles -> H2D -> factor -> D2H lower triangle
    e2e = None
    if args.e2e_steps > 0:
        # every step factors A itself: the pinned buffer is refilled from the
        # device copy of A between steps (outside the timed calls)
        host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        hnp = host.numpy().T  # Fortran view of the column-major bytes
        l = None
        torch.cuda.empty_cache()
        host.copy_(a)
        st_h = plan.factor_host(hnp)  # warm (allocates the staging buffer)
        if st_h.status != "ok":
            raise SystemExit(f"e2e factorization failed: {st_h.status} {st_h.detail}")
        e2e_s = 0.0
        for _ in range(args.e2e_steps):
            host.copy_(a)
            barrier()
            t0 = time.perf_counter()
            st_h = plan.factor_host(hnp)
            e2e_s += time.perf_counter() - t0
            if st_h.status != "ok":
                raise SystemExit(f"e2e factorization failed: {st_h.status} {st_h.detail}")
        barrier()
        if ws > 1:
            e2e_s = allreduce_max(e2e_s, shared)
        # lower triangle in leaf-column strips (the diagonal leaf squares whole),
        # both directions (Engine::enqueue_host)
        h2d = sum((n - j0) * min(b, n - j0) for j0 in range(0, n, b)) * 8
        d2h = h2d
        e2e = {"value": ws * args.e2e_steps * flops / e2e_s / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "status": st_h.status,
               "note": "each step: tc_potrf_host on pinned host doubles holding A (refilled between steps, "
                       "untimed), H2D + factor + D2H of the lower triangle inside the timed call"}

    # C4: a batch of independent N=16384 systems (POTRF + POTRS), sharded
    # across the ranks with no data-path collective
    # release the C3 plan (level buffers, staging copy) and matrices first
    import gc
    plan = a = l = host = hnp = None
    gc.collect()
    torch.cuda.empty_cache()
    c4 = None
    if args.c4_count > 0:
        from paper_2601_08082_b200.batch import run_batch_on_rank
        if ws > 1:
            dist.barrier()
        local, tot, fl = run_batch_on_rank(args.c4_count, args.c4_n, b, CFG, seed0=1000, concurrency=args.c4_conc,
                                           world=ws, rank=rank, in_flight=2 * args.c4_conc)
        c4 = {"workload": f"C4: {args.c4_count} x N={args.c4_n} b={b} {CFG} POTRF+POTRS (1 RHS), sharded over "
                          f"{ws} rank(s), {args.c4_conc} plans per GPU",
              "value": tot.systems * fl / (tot.device_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
              "solves_per_s": tot.systems / (tot.device_ms * 1e-3), "systems": tot.systems, "failed": tot.failed,
              "ms_max_over_ranks": tot.device_ms, "worst_solve_residual": tot.worst_residual,
              "potrs_ms": tot.solve_ms,
              # POTRS reads L twice (forward + backward sweep): n(n+1) * 8 bytes per system and RHS
              "potrs_gbs": (tot.systems * args.c4_n * (args.c4_n + 1) * 8 / (tot.solve_ms * 1e-3) / 1e9
                            if tot.solve_ms > 0 else None),
              "potrs_gbs_note": "algorithmic bytes n(n+1)*8 per system / batched solve phase device time "
                                "(max over ranks)",
              "data": "spd_generate(16384, 1000 + k), bit-identical (mt19937_64 stream), b = A * ones"}

    # C5: one factorization split over the ranks (NCCL broadcast of L11,
    # all-reduce of the panel alpha, all-gather of the solved panel), at the
    # C3 size so it compares with the single-GPU value above
    c5 = None
    if ws > 1 and args.c5_n > 0 and not shared:
        from paper_2601_08082_b200.distributed import potrf_top_split, synthetic_pieces
        a11, a21, a22, l22 = synthetic_pieces(args.c5_n, b, SEED, ws, rank)
        cache = {}
        times = []
        for it in range(3):  # the first call builds the plans
            res = potrf_top_split(args.c5_n, b, CFG, a11=a11.clone() if a11 is not None else None,
                                  a21_rows=a21.clone(), a22_rows=a22.clone(), l22=l22, cache=cache)
            times.append(allreduce_max(res.device_ms, shared))
        ms5 = min(times[1:])
        c5 = {"workload": f"C5-style: one N={args.c5_n} factorization, top TRSM/SYRK row-split over {ws} GPUs, "
                          f"L11 broadcast + alpha all-reduce + panel all-gather over NCCL",
              "value": potrf_flops(args.c5_n) / (ms5 * 1e-3) / 1e12, "unit": "TFLOP/s", "ms": ms5,
              "status": res.status, "scaling": "strong",
              "data": "device-generated SPD of spd_generate's distribution"}
        del a11, a21, a22, l22, cache, res
        torch.cuda.empty_cache()

    variants = None
    if args.variants and rank == 0:
        variants = run_variants(args, tc, torch)

    cpu = None
    if rank == 0 and ws == 1 and args.cpu_n > 0:
        cpu = cpu_baseline_sample(args)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f16 tensor-core (FP32 acc) / f32 / f64 per precision tree",
                "data": "synthetic: spd_generate(65536, 42 + rank), bit-identical to analysis.cpp:12-28",
                "config": {"workload": f"C3: N={n} b={b} {CFG}, quantize on, one factorization per step",
                           "ranks_per_gpu": (ws + ndev - 1) // ndev,
                           "n": n, "b": b, "precision_tree": CFG,
                           "parallelism": f"independent systems x{ws}" if ws > 1 else "single",
                           "l2": f"inputs ({n * n * 8 / 1e9:.1f} GB) larger than the 126 MB L2; no flush needed"},
                "status": st.status, "rel_error": rel, "digits": -math.log10(rel) if rel > 0 else None,
                "clocks": clk.summary(), "gpu_launches": stats["launches"] * args.steps,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "c4": c4, "c5": c5, "variants": variants,
                "breakdown_ms_serialized": {k: round(v[0], 3) for k, v in sorted(by_type.items(),
                                                                                  key=lambda kv: -kv[1][0])}}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_variants(args, tc, torch):
    """accuracy / speed bounds through the same kernels (north_star): Pure F16
    and the mixed tree on A * 2^-1 (Pure F16 overflows the N=65536 diagonal,
    n + r > 65504; the power-of-two scaling is exact), and
    Pure F64 on A."""
    n, b = args.n, args.b
    out = {}
    for name, cfg, scale in (("mixed_half_scaled", CFG, 0.5), ("pure_f16_half_scaled", "Pure F16", 0.5),
                             ("pure_f64", "Pure F64", 1.0)):
        a = tc.spd_generate_device(n, SEED)
        if scale != 1.0:
            a.mul_(scale)
        l = torch.empty_like(a)
        plan = tc.Plan(n, b, cfg, True)
        st = plan.factor_device(a, l)
        reps = 1 if cfg == "Pure F64" else 3
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            plan.factor_device(a, l, sync=False)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / reps
        st = plan.status()
        rel = tc.factorization_error_device(a, l) if st.status == "ok" else float("nan")
        out[name] = {"config": cfg, "input_scale": scale, "status": st.status, "ms": ms,
                     "tflops": potrf_flops(n) / (ms * 1e-3) / 1e12, "rel_error": rel}
        del a, l, plan
        torch.cuda.empty_cache()
    m, h = out["mixed_half_scaled"], out["pure_f16_half_scaled"]
    out["mixed_vs_pure_f16_throughput"] = h["ms"] / m["ms"]
    out["pure_f16_vs_mixed_error"] = h["rel_error"] / m["rel_error"] if m["rel_error"] > 0 else None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # (not --n: torchrun's own parser would take it for a prefix of --nnodes
    # when this script re-launches itself under torchrun)
    ap.add_argument("--size", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--b", type=int, default=B_DEFAULT)
    ap.add_argument("--e2e-steps", dest="e2e_steps", type=int, default=2)
    ap.add_argument("--cpu-n", dest="cpu_n", type=int, default=1536)
    ap.add_argument("--ref-n", dest="ref_n", type=int, default=1536)
    ap.add_argument("--c4-count", dest="c4_count", type=int, default=64)
    ap.add_argument("--c4-n", dest="c4_n", type=int, default=16384)
    ap.add_argument("--c4-conc", dest="c4_conc", type=int, default=16)
    ap.add_argument("--c5-n", dest="c5_n", type=int, default=65536,
                    help="N of the distributed single factorization run when --gpus > 1 (0: off)")
    ap.add_argument("--no-variants", dest="variants", action="store_false",
                    help="skip the Pure F16 / Pure F64 bound runs (on by default)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this command under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    ws, _, _ = dist_env()
    if args.impl == "ours" and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
