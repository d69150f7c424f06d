"""One model's decode iterations via nova_time_pass (for ncu captures).
python scripts/dec_once.py --model 2b --B 2 --s 0 --iters 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as BN  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="2b")
    ap.add_argument("--B", type=int, default=2)
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--ctx", type=int, default=1334)
    ap.add_argument("--iters", type=int, default=2)
    a = ap.parse_args()
    from synth import Q2B, Q7B
    eng = BN.build_engine(Q2B if a.model == "2b" else Q7B, 0)
    print(eng.time_pass(2, a.s, B=a.B, ctx=a.ctx, iters=a.iters))
    eng.close()


if __name__ == "__main__":
    main()
