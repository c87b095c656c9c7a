"""Interleaved A/B of the prepared-Execute step between library builds (SEL_LIB variants):
each round runs every variant in its own subprocess (same seeded C2-shaped table, several row
counts), so slow drifts of the box hit all variants alike. Prints one JSON line per
(variant, rows) with the median over rounds of each round's median step (CUDA events over
back-to-back graph launches) and the library's per-kernel times.

    python scripts/ab_step.py <rounds> <rows,rows,...> base=<path|-> name=<path>[@KEY=VAL,...] ...
    (a variant's @KEY=VAL pairs are set in its subprocess's environment)
    python scripts/ab_step.py --child <rows,...>        (one measurement, used internally)
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(rows):
    import torch
    sys.path.insert(0, ROOT)
    import paper_1806_08384_b200 as sel
    from selgen import configs, encode
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    out = {}
    for n in rows:
        T = configs.gen_c2(n, device=dev)
        t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
        prog = encode(configs.c2_probes()["listing"], T.types)
        q = t.prepare_execute(prog, project=["A", "C", "D"], max_size=n)
        for _ in range(10):
            q.run()
        torch.cuda.synchronize()
        steps = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(40):
                q.run()
            b.record()
            torch.cuda.synchronize()
            steps.append(a.elapsed_time(b) / 40)
        asteps = []
        if hasattr(q, "_fn_async"):   # the same steps returning at the count (async Execute)
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(40):
                    q.run(wait=False)
                b.record()
                torch.cuda.synchronize()
                asteps.append(a.elapsed_time(b) / 40)
        ctx.enable_timing(True)
        ks = []
        for _ in range(20):
            q.run()
            ks.append(ctx.last_times())
        ctx.enable_timing(False)
        out[n] = {"step": statistics.median(steps),
                  "step_async": statistics.median(asteps) if asteps else None,
                  "count": statistics.median(k[0] for k in ks),
                  "pushdown": statistics.median(k[1] for k in ks)}
        q.release()
        t.release()
        del T
        torch.cuda.empty_cache()
    ctx.close()
    print(json.dumps(out))


def main():
    if sys.argv[1] == "--child":
        child([int(x) for x in sys.argv[2].split(",")])
        return
    rounds = int(sys.argv[1])
    rows = sys.argv[2]
    variants = [a.split("=", 1) for a in sys.argv[3:]]
    res = {name: [] for name, _ in variants}
    for _ in range(rounds):
        for name, spec in variants:
            env = dict(os.environ)
            env.pop("SEL_LIB", None)
            path, _, extra = spec.partition("@")
            if path != "-":
                env["SEL_LIB"] = path
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            r = subprocess.run([sys.executable, __file__, "--child", rows], env=env,
                               capture_output=True, text=True, timeout=600)
            if r.returncode != 0:
                print(json.dumps({"variant": name, "error": r.stderr[-400:]}), flush=True)
                continue
            res[name].append(json.loads(r.stdout.strip().splitlines()[-1]))
    for name, runs in res.items():
        for n in rows.split(","):
            xs = [r[n] for r in runs if n in r]
            if not xs:
                continue
            print(json.dumps({"variant": name, "rows": int(n), "rounds": len(xs),
                              **{k: round(statistics.median(x[k] for x in xs), 4)
                                 for k in ("step", "count", "pushdown")},
                              "step_async": (round(statistics.median(x["step_async"] for x in xs), 4)
                                             if all(x.get("step_async") for x in xs) else None),
                              "step_all": [round(x["step"], 4) for x in xs]}), flush=True)


if __name__ == "__main__":
    main()
