#!/usr/bin/env python
"""A/B kernel variants on one box: bench.py (kernel-only legs) per library variant, alternating.

    python tools/ab_variants.py --config c2 --rounds 2 --variants base seq seqp1 [--out f.jsonl]

`base` is libcqs.so; any other name X loads paper_2604_20819_b200/libcqs_X.so (built with
build(variant=X, defines=[...])) through CQS_LIB.  Each run prints bench.py's value, the attention
kernels' roofline.achieved and the sampled clocks.  Alternating the variants over rounds spreads
box drift (power cap, temperature) over all of them.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--variants", nargs="+", default=["base"])
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    for r in range(args.rounds):
        for v in args.variants:
            env = dict(os.environ)
            if v != "base":
                env["CQS_LIB"] = os.path.join(ROOT, "paper_2604_20819_b200", "libcqs_%s.so" % v)
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", args.config,
                   "--steps", str(args.steps), "--warmup", "3", "--no-cpu", "--no-e2e", "--no-bwd",
                   "--no-budget"]
            p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
            row = {"variant": v, "round": r, "config": args.config}
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
                row.update(value=d["value"], kernel=d["roofline"]["achieved"],
                           sm_mhz=d["clocks"].get("sm_mhz"), reasons=d["clocks"].get("reasons"),
                           power_w_max=d["clocks"].get("power_w_max"))
            except Exception as ex:
                row["error"] = "%s | %s" % (ex, (p.stderr or "")[-600:])
            print(json.dumps(row), flush=True)
            rows.append(row)
    if args.out:
        with open(args.out, "a") as f:
            for row in rows:
                f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
