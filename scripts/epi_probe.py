"""GEMM epilogue cost probe: one shape, every epilogue (graph-timed like kbench)."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
from paper_2509_21301_b200 import ops as O
from kbench import timeit, rnd
for (M, N, K) in [(4888, 1280, 1280), (4888, 1280, 5120), (4888, 5120, 1280), (1286, 3584, 18944)]:
    A = rnd((M, K)); W = rnd((N, K), scale=K ** -0.5); bias = rnd((N,), scale=0.1)
    for epi, name in [(O.EPI_BF16, "bf16"), (O.EPI_BF16_QGELU, "qgelu"), (O.EPI_F32_STORE, "f32"), (O.EPI_F32_RESID, "resid")]:
        C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (O.EPI_F32_RESID, O.EPI_F32_STORE) else torch.bfloat16)
        ms = timeit(lambda i: O.nova_op_gemm(A, W, C, bias, M, N, K, epi), 20, 1)
        print(json.dumps({"M": M, "N": N, "K": K, "epi": name, "us": round(ms * 1e3, 1),
                          "TFLOP/s": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
