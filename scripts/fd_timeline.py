"""Fused decode kernel phase timeline (NOVA_DEC_FUSED_DBG=4): per phase, when CTA 0 saw the
barrier, when the last CTA arrived.  python scripts/fd_timeline.py --model 2b --B 2 --s 0"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NOVA_DEC_FUSED_DBG"] = os.environ.get("NOVA_DEC_FUSED_DBGX", "4")
import bench as BN  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="2b")
    ap.add_argument("--B", type=int, default=2)
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--ctx", type=int, default=1334)
    a = ap.parse_args()
    from synth import Q2B, Q7B
    sh = Q2B if a.model == "2b" else Q7B
    eng = BN.build_engine(sh, 0)
    ms = eng.time_pass(2, a.s, B=a.B, ctx=a.ctx, iters=5)[0]
    L = sh.llm_layers
    raw = np.frombuffer(eng.debug_read_buffer("dec_dbg", 8 * 2048), dtype=np.uint64).astype(np.int64)
    t = raw[:3 * (5 * L + 2)].reshape(-1, 3)
    mk = raw[1024:1024 + 64].reshape(8, 8)
    t0 = t[0, 0]
    names = ["embed"] + [f"{n}{l}" for l in range(L) for n in ("qkv", "attn", "o", "gu", "down")] + ["lm"]
    rows = []
    for ph in range(5 * L + 2):
        seen = (t[ph, 0] - t0) / 1e3 if ph > 0 else 0.0
        last = (t[ph, 1] - t0) / 1e3
        rows.append((names[ph], round(seen, 2), round(last, 2)))
    kinds = {}
    for ph in range(1, 5 * L + 2):
        k = names[ph].rstrip("0123456789")
        span = rows[ph][2] - rows[ph][1]          # barrier seen -> last arrival
        lat = rows[ph][1] - rows[ph - 1][2]       # previous last arrival -> barrier seen by CTA 0
        kinds.setdefault(k, [0.0, 0.0, 0])
        kinds[k][0] += span
        kinds[k][1] += lat
        kinds[k][2] += 1
    print(json.dumps({"model": sh.name, "B": a.B, "s": a.s, "ms": round(ms, 3), "total_us": rows[-1][2],
                      "per_kind_us": {k: {"span": round(v[0], 1), "barrier_lat": round(v[1], 1), "n": v[2]}
                                      for k, v in kinds.items()},
                      "first_layers": rows[:12],
                      "last_layer_milestones_us": {
                          kn: [round((mk[k, m] - t[phs, 0]) / 1e3, 2) for m in range(5) if mk[k, m] > 0]
                          for kn, k, phs in [("qkv", 1, 5 * L - 4), ("attn", 2, 5 * L - 3), ("o", 3, 5 * L - 2),
                                             ("gu", 4, 5 * L - 1), ("down", 5, 5 * L), ("lm", 6, 5 * L + 1)]},
                      "last_layer_span_us": {n: round((t[ph, 1] - t[ph, 0]) / 1e3, 2) for n, ph in
                                             [("qkv", 5 * L - 4), ("attn", 5 * L - 3), ("o", 5 * L - 2), ("gu", 5 * L - 1),
                                              ("down", 5 * L), ("lm", 5 * L + 1)]}}))
    eng.close()


if __name__ == "__main__":
    main()
