"""Timeline of the last gemv_umma launch with N == NOVA_UMMA_TRACE_N inside decode iterations on a
green-context partition (library built with -DNOVA_UMMA_TRACE).

    NOVA_UMMA_TRACE_N=17920 python scripts/umma_trace_pass.py --model 2b --s 24 --B 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import bench as BN  # noqa: E402
from umma_trace import read_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="2b")
    ap.add_argument("--B", type=int, default=2)
    ap.add_argument("--s", type=int, nargs="*", default=[24])
    ap.add_argument("--ctx", type=int, default=1334)
    a = ap.parse_args()
    from synth import Q2B, Q7B
    eng = BN.build_engine(Q2B if a.model == "2b" else Q7B, 0)
    eng.time_pass(2, 0, B=a.B, ctx=a.ctx, iters=2)
    for s in a.s:
        ms = eng.time_pass(2, s, B=a.B, ctx=a.ctx, iters=3)[0]
        read_trace({"model": a.model, "s": s, "B": a.B, "N": int(os.environ.get("NOVA_UMMA_TRACE_N", -1)),
                    "iter_ms": round(ms, 3)})
    eng.close()


if __name__ == "__main__":
    main()
