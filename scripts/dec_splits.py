"""Decode iteration time (ms) on green-context partitions s (0 = whole GPU) via nova_time_pass.
    python scripts/dec_splits.py --model 2b --B 2 [--splits 0 24 32 48 64]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as BN  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="2b")
    ap.add_argument("--B", type=int, nargs="*", default=[2])
    ap.add_argument("--ctx", type=int, default=1334)
    ap.add_argument("--splits", type=int, nargs="*", default=[0, 24, 32, 48, 64])
    a = ap.parse_args()
    from synth import Q2B, Q7B
    eng = BN.build_engine(Q2B if a.model == "2b" else Q7B, 0)
    eng.time_pass(2, 0, B=2, ctx=a.ctx, iters=3)
    for B in a.B:
        out = {s: round(eng.time_pass(2, s, B=B, ctx=a.ctx, iters=8)[0], 3) for s in a.splits}
        print(json.dumps({"model": a.model, "B": B, "ms": out, "env": {k: v for k, v in os.environ.items()
                                                                       if k.startswith("NOVA_")}}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
