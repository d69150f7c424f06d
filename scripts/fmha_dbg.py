import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21301_b200 import ops as O
from paper_2509_21301_b200._lib import lib
S, H, KV, hd, causal = (int(x) for x in sys.argv[1:6])
qkv = torch.randn(S, (H + 2 * KV) * hd, device="cuda").bfloat16()
out = torch.empty(S, H * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    O.nova_op_flash_attn(qkv, out, S, H, KV, hd, causal)
torch.cuda.synchronize()
buf = np.zeros((16, 512), np.int64)
f = lib().nova_op_fmha_debug
f.argtypes = [ctypes.c_void_p]
print("rc", f(buf.ctypes.data))
t0 = buf[0, 0]
names = ["A.pre", "A.s_ok", "A.turn_ok", "A.done", "B.pre", "B.s_ok", "B.turn_ok", "B.done",
         "M.top", "M.v_ok", "M.pA_ok", "M.k_ok", "M.A_iss", "M.pB_ok", "M.B_iss", "-"]
for g in range(0, 24):
    ev = sorted([(buf[e, g] - t0, names[e]) for e in range(15)])
    print(g, " ".join(f"{n}={t}" for t, n in ev))
d = buf[:, 10:70]
print("per-tile period A", np.diff(d[3]).mean(), "B", np.diff(d[7]).mean())
print("A wait S", (d[1] - d[0]).mean(), "A wait turn", (d[2] - d[1]).mean(), "A exp+store", (d[3] - d[2]).mean())
print("B wait S", (d[5] - d[4]).mean(), "B wait turn", (d[6] - d[5]).mean(), "B exp+store", (d[7] - d[6]).mean())
print("A done->next pre", (d[0, 1:] - d[3, :-1]).mean())
