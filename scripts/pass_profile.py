"""Solo pass timings at the cfg-3 shapes (7B), optionally bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off --metrics gpu__time_duration.sum` lists exactly the kernels of one
pass (warm-up pass + timed pass).  Prints one JSON object per pass with the event-timed ms and the
algorithmic work.

    python scripts/pass_profile.py [--stage vit|pre|dec|all] [--profile] [--iters N] [--B 2 --ctx 1334]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--stage", default="all")
    p.add_argument("--profile", action="store_true")
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--B", type=int, default=2)
    p.add_argument("--ctx", type=int, default=1334)
    p.add_argument("--split", type=int, default=0)
    p.add_argument("--model", default="7b")
    a = p.parse_args()
    from bench import build_engine
    from synth import Q7B, Q2B
    shape = Q7B if a.model == "7b" else Q2B
    eng = build_engine(shape, 0)
    stages = ["vit", "pre", "dec"] if a.stage == "all" else a.stage.split(",")
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6548.0, "bf16_tflops_sustained": 1366.0}
    D, F, V = shape.llm_dim, shape.llm_ffn, shape.vocab
    for st in stages:
        sid = {"vit": 0, "pre": 1, "dec": 2}[st]
        if a.profile:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
            eng.time_pass(sid, a.split, 52, 94, 64, B=a.B, ctx=a.ctx, iters=1)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            continue
        ms = eng.time_pass(sid, a.split, 52, 94, 64, B=a.B, ctx=a.ctx, iters=a.iters)[0]
        rec = {"stage": st, "split": a.split, "ms": round(ms, 4)}
        if st == "vit":
            N = 52 * 94
            fl = 32 * (2 * N * (1280 * 3840 + 1280 ** 2 + 2 * 1280 * 5120) + 4 * N * N * 1280) + \
                2 * N * 1176 * 1280 + 2 * (N // 4) * (5120 ** 2 + 5120 * D)
            rec.update(tflops=round(fl / ms / 1e9, 1), frac=round(fl / ms / 1e9 / pk["bf16_tflops_sustained"], 4))
        elif st == "pre":
            S, H, KV, hd = 1222 + 64, shape.llm_heads, shape.llm_kv_heads, shape.head_dim
            fl = shape.llm_layers * (2 * S * (D * (D + 2 * KV * hd) + D * D + 3 * D * F) + 2 * S * S * H * hd) + 2 * D * V
            rec.update(tflops=round(fl / ms / 1e9, 1), frac=round(fl / ms / 1e9 / pk["bf16_tflops_sustained"], 4))
        else:
            W = shape.llm_layers * 2 * (D * (D + 2 * shape.llm_kv_heads * shape.head_dim) + D * D + 3 * D * F) + 2 * D * V
            kv = a.B * (a.ctx + 1) * shape.llm_layers * 2 * shape.llm_kv_heads * shape.head_dim * 2
            rec.update(gbs=round((W + kv) / ms / 1e6, 1), frac=round((W + kv) / ms / 1e6 / pk["hbm_gbs"], 4),
                       B=a.B, ctx=a.ctx)
        print(json.dumps(rec), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
