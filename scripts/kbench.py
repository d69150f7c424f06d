"""Per-kernel roofline micro-benchmark at the 7B / ViT shapes, through
the op-level C ABI (include/nova_ops.h).  Each kernel is timed with CUDA events on the stream it
is launched on, over rotating weight copies larger than L2 (126 MB) so the weight stream comes
from HBM.  Prints one JSON object per kernel: achieved GB/s or TFLOP/s and the fraction of the
measured peak (MEASURED_PEAKS.json).

    python scripts/kbench.py [--only gemv|gemm|attn|dattn] [--iters N]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_21301_b200 import ops as O  # noqa: E402

PK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
HBM, TFL = PK["hbm_gbs"], PK["bf16_tflops"]


def timeit(fn, iters, rot):
    """ms per call: `iters` back-to-back calls captured in one CUDA graph (no Python/launch
    overhead between kernels, PDL edges kept), replayed after a warm-up, CUDA events."""
    for i in range(3):
        fn(i % rot)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i % rot)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * iters)


def rnd(shape, dtype=torch.bfloat16, scale=1.0):
    return (torch.randn(shape, device="cuda") * scale).to(dtype)


def bench_gemv(iters):
    D, F, V, H, KV, hd = 3584, 18944, 152064, 28, 4, 128
    shapes = [("qkv", (H + 2 * KV) * hd, D, O.EPI_BF16, False), ("o", D, H * hd, O.EPI_F32_RESID, False),
              ("gate_up", 2 * F, D, O.EPI_BF16_SILUMUL, False), ("down", D, F, O.EPI_F32_RESID, False),
              ("lm_head", V, D, O.EPI_F32_STORE, True)]
    for name, N, K, epi, xf in shapes:
        wbytes = N * K * 2
        rot = max(1, int(300e6 // wbytes) + 1)
        Ws = [rnd((N, K), scale=K ** -0.5) for _ in range(rot)]
        for B in (1, 4, 8, 16):
            X = rnd((B, K)) if not xf else torch.randn(B, K, device="cuda")
            nout = N // 2 if epi == O.EPI_BF16_SILUMUL else N
            Y = torch.zeros(B, nout, device="cuda", dtype=torch.bfloat16 if epi in (O.EPI_BF16, O.EPI_BF16_SILUMUL)
                            else torch.float32)
            byt = wbytes + B * K * (4 if xf else 2) + B * nout * (8 if epi == O.EPI_F32_RESID else 4)
            variants = [("gemv", lambda i: O.nova_op_gemv(X, Ws[i], Y, None, N, K, B, epi))]
            if not xf:
                variants.append(("gemv_tma", lambda i: O.nova_op_gemv_tma(X, Ws[i], Y, None, N, K, B, epi)))
            if name in ("qkv", "gate_up", "lm_head"):   # RMSNorm applied on load from the f32 residual rows
                Xf = torch.randn(B, K, device="cuda")
                gam = torch.ones(K, device="cuda", dtype=torch.bfloat16)
                xm = O.XM_NORM_F32 if xf else O.XM_NORM_BF16
                variants.append(("gemv_norm", lambda i: O.nova_op_gemv_fused(Xf, xm, Ws[i], Y, None, N, K, B, epi,
                                                                             gamma=gam, eps=1e-6)))
            for kname, fn in variants:
                ms = timeit(fn, iters, rot)
                gbs = byt / ms / 1e6
                print(json.dumps({"kernel": kname, "shape": name, "N": N, "K": K, "B": B,
                                  "us": round(ms * 1e3, 2), "GB/s": round(gbs, 1),
                                  "frac_hbm": round(gbs / HBM, 3)}), flush=True)
        del Ws


GEMM_MODES = [0]


def bench_gemm(iters):
    cases = [("vit_qkv", 4888, 3840, 1280, O.EPI_BF16), ("vit_proj", 4888, 1280, 1280, O.EPI_F32_RESID),
             ("vit_fc1", 4888, 5120, 1280, O.EPI_BF16_QGELU), ("vit_fc2", 4888, 1280, 5120, O.EPI_F32_RESID),
             ("vit_fc1_7920", 7920, 5120, 1280, O.EPI_BF16_QGELU),
             ("pre_qkv", 1286, 4608, 3584, O.EPI_BF16), ("pre_gate_up", 1286, 37888, 3584, O.EPI_BF16_SILUMUL),
             ("pre_down", 1286, 3584, 18944, O.EPI_F32_RESID), ("sq8192", 8192, 8192, 8192, O.EPI_BF16)]
    for name, M, N, K, epi in cases:
        A = rnd((M, K))
        W = rnd((N, K), scale=K ** -0.5)
        bias = rnd((N,), scale=0.1) if epi != O.EPI_BF16_SILUMUL else None
        nout = N // 2 if epi == O.EPI_BF16_SILUMUL else N
        C = torch.zeros(M, nout, device="cuda", dtype=torch.float32 if epi == O.EPI_F32_RESID else torch.bfloat16)
        for mode in GEMM_MODES:
            prev = O.nova_op_gemm_mode(mode)
            tile = O.nova_op_gemm_config(M, N, K)
            for sms in ((148, 100) if mode == 0 else (148,)):
                if tile < 0:
                    continue
                ms = timeit(lambda i: O.nova_op_gemm(A, W, C, bias, M, N, K, epi, max_ctas=sms), iters, 1)
                tf = 2.0 * M * N * K / ms / 1e9
                print(json.dumps({"kernel": "gemm_tc", "shape": name, "M": M, "N": N, "K": K, "ctas": sms,
                                  "mode": mode, "tile": tile, "us": round(ms * 1e3, 1), "TFLOP/s": round(tf, 1),
                                  "frac_tensor": round(tf / TFL, 3)}), flush=True)
            O.nova_op_gemm_mode(prev)


def bench_attn(iters):
    for name, S, H, KV, hd, causal in [("vit_4888", 4888, 16, 16, 80, 0), ("vit_7920", 7920, 16, 16, 80, 0),
                                        ("pre_1286", 1286, 28, 4, 128, 1), ("pre_2044", 2044, 28, 4, 128, 1),
                                        ("pre2b_1286", 1286, 12, 2, 128, 1)]:
        qkv = rnd((S, (H + 2 * KV) * hd))
        out = torch.empty(S, H * hd, device="cuda", dtype=torch.bfloat16)
        fl = (2.0 if causal else 4.0) * S * S * hd * H
        for kname, fn in [("flash_attn_tc", O.nova_op_flash_attn), ("flash_attn_mma", O.nova_op_flash_attn_mma)]:
            ms = timeit(lambda i: fn(qkv, out, S, H, KV, hd, causal), iters, 1)
            tf = fl / ms / 1e9
            print(json.dumps({"kernel": kname, "shape": name, "us": round(ms * 1e3, 1), "TFLOP/s": round(tf, 1),
                              "frac_tensor": round(tf / TFL, 3)}), flush=True)


def bench_dattn(iters):
    H, KV, hd, L = 28, 4, 128, 1
    for B, ctx in [(1, 1334), (2, 1334), (4, 1334), (8, 1334), (16, 1334), (16, 2047)]:
        pages = (ctx + 64) // 64
        n_pages = B * pages
        pool = rnd((L, n_pages, 2, KV, 64, hd))
        bt = torch.arange(n_pages, dtype=torch.int32, device="cuda").view(B, pages)
        rows = torch.tensor([[b, ctx, 0, 0] for b in range(B)], dtype=torch.int32, device="cuda")
        qkv = rnd((B, (H + 2 * KV) * hd))
        out = torch.empty(B, H * hd, device="cuda", dtype=torch.bfloat16)
        ws = torch.empty(B * H * ((ctx + 128) // 128 + 1) * 4 * (hd + 2), device="cuda")
        tk = torch.zeros(B * KV, dtype=torch.int32, device="cuda")
        ms = timeit(lambda i: O.nova_op_decode_attn(qkv, out, pool, 0, n_pages, H, KV, hd, bt, rows, B, ctx, ws, tk),
                    iters, 1)
        byt = B * (ctx + 1) * 2 * KV * hd * 2
        print(json.dumps({"kernel": "decode_attn", "B": B, "ctx": ctx, "us": round(ms * 1e3, 2),
                          "GB/s": round(byt / ms / 1e6, 1), "frac_hbm": round(byt / ms / 1e6 / HBM, 3)}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--gemm-modes", default="0", help="comma list: 0 auto, 1 single-CTA, 2 pair, or a tile code "
                    "pair*1000+BN (e.g. 1224)")
    a = ap.parse_args()
    GEMM_MODES[:] = [int(x) for x in a.gemm_modes.split(",")]
    for nm, fn in [("gemv", bench_gemv), ("gemm", bench_gemm), ("attn", bench_attn), ("dattn", bench_dattn)]:
        if a.only in (None, nm):
            fn(a.iters)
