"""Decode pass on an s-SM partition: solo (front idle) vs co-run with the ViT on the rest.

    python scripts/dec_slice_probe.py [--model 2b|7b] [--B 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as BN  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="2b", choices=["2b", "7b"])
    ap.add_argument("--B", type=int, default=2)
    a = ap.parse_args()
    from synth import Q7B, Q2B
    shape = Q2B if a.model == "2b" else Q7B
    eng = BN.build_engine(shape, 0)
    total, g, nsplit = eng.query_sms()
    eng.time_pass(2, 0, B=a.B, ctx=1334, iters=3)
    full = eng.time_pass(2, 0, B=a.B, ctx=1334, iters=10)[0]
    print(json.dumps({"model": shape.name, "B": a.B, "full_ms": round(full, 3)}), flush=True)
    for s in [g * k for k in range(1, nsplit + 1)]:
        solo = eng.time_pass(2, s, B=a.B, ctx=1334, iters=5)[0]
        f, co = eng.time_pass(0, s, 52, 94, B=a.B, ctx=1334, corun=1, iters=2)
        print(json.dumps({"s": s, "dec_solo_ms": round(solo, 3), "dec_corun_vit_ms": round(co, 3),
                          "vit_corun_ms": round(f, 3)}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
