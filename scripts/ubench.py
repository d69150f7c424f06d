"""Decode-linear micro-benchmark: the mma.sync TMA GEMV (nova_op_gemv_stream) vs the tcgen05 GEMV
(nova_op_gemv_umma) at the 2B / 7B decode shapes, per grid budget (max_ctas; without a green context
the CTAs still spread over all SMs) and batch.  Weights rotate over copies > L2.  JSON lines.

    python scripts/ubench.py [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from kbench import timeit, rnd  # noqa: E402
from paper_2509_21301_b200 import ops as O  # noqa: E402

SHAPES = {"2b_gu": (17920, 1536, O.EPI_BF16_SILUMUL), "2b_down": (1536, 8960, O.EPI_F32_RESID),
          "2b_o": (1536, 1536, O.EPI_F32_RESID), "2b_lm": (151936, 1536, O.EPI_F32_ARGMAX),
          "7b_gu": (37888, 3584, O.EPI_BF16_SILUMUL), "7b_down": (3584, 18944, O.EPI_F32_RESID)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    for name, (N, K, epi) in SHAPES.items():
        if a.only and a.only not in name:
            continue
        rot = max(2, int(300e6 // (N * K * 2)) + 1)
        Wbs = []
        for _ in range(rot):
            W = rnd((N, K), scale=K ** -0.5)
            Wb = torch.empty_like(W)
            O.nova_op_block_weights(W, Wb, N, K)
            Wbs.append(Wb)
            del W
        for B in (2, 16):
            X = rnd((2 * B, K))
            nout = N // 2 if epi == O.EPI_BF16_SILUMUL else N
            Y = torch.zeros(B, nout, dtype=torch.bfloat16 if epi == O.EPI_BF16_SILUMUL else torch.float32,
                            device="cuda")
            keys = torch.zeros(B, dtype=torch.int64, device="cuda")
            for ctas in (148, 64, 32, 24):
                row = {"op": name, "B": B, "ctas": ctas}
                for kname, fn in (("tma", O.nova_op_gemv_stream), ("umma", O.nova_op_gemv_umma)):
                    xlo = X[B:] if epi == O.EPI_F32_ARGMAX else None

                    def call(i, fn=fn, xlo=xlo):
                        fn(X[:B], Wbs[i], Y, None, N, K, B, epi, X_lo=xlo, keys=keys, max_ctas=ctas)
                    ms = timeit(call, a.iters, rot)
                    row[kname + "_us"] = round(ms * 1e3, 2)
                    row[kname + "_GBs"] = round(N * K * 2 / (ms / 1e3) / 1e9, 1)
                print(json.dumps(row), flush=True)
        del Wbs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
