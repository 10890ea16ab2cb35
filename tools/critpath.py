"""Development tool: per-op serialized device times of one factorization and
the DAG's critical path (longest dependency chain weighted by those times).

    python tools/critpath.py --n 65536            # summary by op type
    python tools/critpath.py --n 65536 --ncu-pick # k_gemm_tc launch index of the largest tc16 op

The critical path bounds what stream/graph concurrency can reach; the gap
between it and the graph-replay time is scheduling loss.
"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
    ap.add_argument("--ncu-pick", action="store_true")
    ap.add_argument("--pick-n", type=int, default=0, help="with --ncu-pick: the largest tc16 op whose first problem has this n")
    ap.add_argument("--pick-class", default="tc16", help="with --ncu-pick: tc16 or tc32")
    ap.add_argument("--profile-only", action="store_true", help="one serialized run (for ncu)")
    ap.add_argument("--json", default="")
    ap.add_argument("--opt", action="append", default=[], help="plan option key=value (repeatable)")
    args = ap.parse_args()
    plan = tc.Plan(args.n, args.b, args.cfg)
    for kv in args.opt:
        k, v = kv.split("=")
        plan.set_option(k, int(v))
    nops = plan.stats()["ops"]
    infos = [plan.op_info(i) for i in range(nops)]
    if args.ncu_pick:
        # launch order of the serialized profile run == op order; the index
        # counts every k_gemm_tc launch (both operand kinds match the name)
        # (k_gemm_tc<0> and <1> are separate kernels for ncu's -k regex:
        # count launches of the picked class only)
        best, best_i, idx = -1.0, -1, 0
        for i, inf in enumerate(infos):
            if inf["type"] == "gemm" and inf["gclass"] == args.pick_class:
                ok = not args.pick_n or plan.op_probs(i)[0]["n"] == args.pick_n
                if ok and inf["flops"] > best:
                    best, best_i = inf["flops"], idx
                idx += 1
        print(best_i)
        return
    a = tc.spd_generate_device(args.n, 42)
    l = torch.empty_like(a)
    if args.profile_only:
        plan.profile(a, l)
        torch.cuda.synchronize()
        return
    st = plan.factor_device(a, l)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    plan.factor_device(a, l, sync=False)
    ev1.record()
    torch.cuda.synchronize()
    graph_ms = ev0.elapsed_time(ev1)
    op_ms = plan.profile(a, l)
    deps = [plan.op_deps(i) for i in range(nops)]
    finish = [0.0] * nops
    via = [-1] * nops
    for i in range(nops):
        s, v = 0.0, -1
        for d in deps[i]:
            if finish[d] > s:
                s, v = finish[d], d
        finish[i] = s + op_ms[i]
        via[i] = v
    end = max(range(nops), key=lambda i: finish[i])
    path = []
    i = end
    while i >= 0:
        path.append(i)
        i = via[i]
    path.reverse()

    def key(inf):
        return inf["type"] + ("/" + inf["gclass"] if inf["gclass"] else "") + "/L%d" % inf["level"]

    tot, crit = {}, {}
    for i in range(nops):
        e = tot.setdefault(key(infos[i]), [0.0, 0, 0.0])
        e[0] += op_ms[i]
        e[1] += 1
        e[2] += infos[i]["flops"]
    for i in path:
        e = crit.setdefault(key(infos[i]), [0.0, 0])
        e[0] += op_ms[i]
        e[1] += 1
    out = {"n": args.n, "cfg": args.cfg, "status": st.status, "graph_ms": graph_ms, "serial_ms": sum(op_ms),
           "critical_ms": finish[end], "critical_ops": len(path),
           "tflops_graph": tc.potrf_flops(args.n) / graph_ms / 1e9}
    print(json.dumps(out))
    print("%-26s %10s %6s %9s | %10s %6s" % ("op", "serial ms", "n", "TF/s", "crit ms", "n"))
    for k, (t, c, f) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        ct, cc = crit.get(k, [0.0, 0])
        print("%-26s %10.3f %6d %9.1f | %10.3f %6d" % (k, t, c, f / t / 1e9 if t else 0, ct, cc))
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"summary": out, "ops": [dict(infos[i], ms=op_ms[i], deps=deps[i]) for i in range(nops)],
                       "path": path}, f)


if __name__ == "__main__":
    main()
