"""Per-CTA timeline of one gemv_umma launch (library built with -DNOVA_UMMA_TRACE).

    python scripts/umma_trace.py N K epi ctas [B]

Prints, over the CTAs: launch skew (t0), pdl wait (t1 - t0), first stage landed (t2 - t1), weight
stream (t3 - t2), epilogue lag after the last stage (t4 - t3), last ticket (t5), and the critical CTA.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_21301_b200 import ops as O  # noqa: E402
from paper_2509_21301_b200._lib import lib  # noqa: E402



def read_trace(meta):
    n = 2048
    buf = (ctypes.c_ulonglong * (n * 8))()
    f = lib().nova_debug_umma_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert f(ctypes.addressof(buf), n) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    ok = (t[:, 0] > 0) & (t[:, 4] >= t[:, 0])
    ok &= t[:, 0] >= t[ok, 0].max() - 500_000  # entries of earlier, larger grids are stale
    t = t[ok]
    g = int(ok.sum())
    t0 = t[:, 0].min()
    rel = (t[:, :6] - t0) / 1e3  # us
    rng = [(int(v) >> 32, int(v) & 0xFFFFFFFF) for v in t[:, 6]]
    crit = int(np.argmax(t[:, 4]))

    def q(x):
        return [round(float(np.percentile(x, p)), 2) for p in (0, 50, 90, 100)]

    meta.update({"grid": g, "env": {k: v for k, v in os.environ.items() if k.startswith("NOVA_")},
                 "span_us": round(float(rel[:, 4].max()), 2),
                 "t0_start": q(rel[:, 0]), "pdl_wait": q(rel[:, 1] - rel[:, 0]),
                 "first_stage": q(rel[:, 2] - rel[:, 1]), "stream": q(rel[:, 3] - rel[:, 2]),
                 "epi_lag": q(rel[:, 4] - rel[:, 3]), "end": q(rel[:, 4]),
                 "critical": {"cta": crit, "rem_start_n": rng[crit], "t": [round(float(x), 2) for x in rel[crit]]}})
    print(json.dumps(meta), flush=True)


def main():
    N, K, epi, ctas = (int(x) for x in sys.argv[1:5])
    B = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    copies = []
    for _ in range(4):
        W = (torch.randn(N, K, device="cuda") * K ** -0.5).bfloat16()
        Wb = torch.empty_like(W)
        O.nova_op_block_weights(W, Wb, N, K)
        copies.append(Wb)
        del W
    X = torch.randn(2 * B, K, device="cuda").bfloat16()
    nout = N // 2 if epi == O.EPI_BF16_SILUMUL else N
    Y = torch.zeros(B, nout, dtype=torch.bfloat16 if epi == O.EPI_BF16_SILUMUL else torch.float32, device="cuda")
    keys = torch.zeros(B, dtype=torch.int64, device="cuda")
    xlo = X[B:] if epi == O.EPI_F32_ARGMAX else None
    for i in range(6):
        O.nova_op_gemv_umma(X[:B], copies[i % 3], Y, None, N, K, B, epi, X_lo=xlo, keys=keys, max_ctas=ctas)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.fill_(1)
    torch.cuda.synchronize()
    O.nova_op_gemv_umma(X[:B], copies[3], Y, None, N, K, B, epi, X_lo=xlo, keys=keys, max_ctas=ctas)
    torch.cuda.synchronize()
    read_trace({"N": N, "K": K, "epi": epi, "ctas": ctas, "B": B, "splits": O.nova_op_gemv_umma_splits(N, K, epi)})


if __name__ == "__main__":
    main()
