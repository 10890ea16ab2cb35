"""Quick device probe: per-size timing + per-op profile (development tool)."""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_08082_b200 as tc  # noqa: E402


def gen_dev(n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    a = (r + r.T) * 0.5
    a.diagonal().add_(float(n))
    return a.contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[4096, 16384])
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--use_tc", type=int, default=1)
    ap.add_argument("--streams", type=int, default=0)
    ap.add_argument("--err", action="store_true")
    args = ap.parse_args()
    for n in args.n:
        a = gen_dev(n)
        l = torch.empty_like(a)
        plan = tc.Plan(n, args.b, args.cfg, use_tc=bool(args.use_tc), n_streams=args.streams)
        t0 = time.time()
        st = plan.factor_device(a, l)
        torch.cuda.synchronize()
        first = time.time() - t0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(args.reps):
            ev0.record()
            plan.factor_device(a, l, sync=False)
            ev1.record()
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        best = min(ms)
        flops = tc.potrf_flops(n)
        out = {"n": n, "cfg": args.cfg, "status": st.status, "detail": st.detail, "first_s": round(first, 3),
               "ms": [round(x, 3) for x in ms], "tflops": round(flops / best / 1e9, 2), "stats": plan.stats()}
        if args.err:
            out["rel_error"] = tc.factorization_error_device(a, l)
        print(json.dumps(out), flush=True)
        if args.profile:
            op_ms = plan.profile(a, l)
            tot = sum(op_ms)
            agg = {}
            for i, t in enumerate(op_ms):
                info = plan.op_info(i)
                key = info["type"] + ("/" + info["gclass"] if info["gclass"] else "") + "/L%d" % info["level"]
                e = agg.setdefault(key, [0.0, 0, 0.0])
                e[0] += t
                e[1] += 1
                e[2] += info["flops"]
            print("profile total %.2f ms (serialized)" % tot)
            for k, (t, c, f) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
                print("  %-28s %9.3f ms %5.1f%%  n=%5d  %8.1f TF/s" % (k, t, 100 * t / tot, c, f / t / 1e9 if t else 0))
        del a, l, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
