"""Partition-policy sweep on one B200 (R12 evidence): profile the co-run curves once,
then replay the same bursty traces (3 seeds per offered load) under adaptive policies with
different SM_min / alpha readings, the static 50/50 split and serial stage execution.

    python scripts/policy_sweep.py [--rho 0.5 0.7] [--seeds 3] [--requests 48]
Prints one JSON line per (rho, policy) with mean-over-seeds max / p99 / mean E2E and req/s.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as BN  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rho", type=float, nargs="*", default=[0.5, 0.7])
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--sm-min", type=int, nargs="*", default=[])
    ap.add_argument("--sm-op", type=int, nargs="*", default=[], help="adaptive SM_op values (both contexts)")
    ap.add_argument("--offload", type=int, default=0, help="K resident ViT layer slots (0 = all resident)")
    ap.add_argument("--floor", type=int, nargs="*", default=[], help="adaptive + offload-aware sm_dv_floor values")
    ap.add_argument("--policies", default="serial,multi_stream", help="baselines to include")
    ap.add_argument("--model", default="7b", choices=["7b", "2b"])
    ap.add_argument("--trace", default="mmpp", choices=["mmpp", "poisson"],
                    help="mmpp: cfg 3 bursty mix; poisson: cfg 2 (52x94 screenshots, prompt 64, gen 48)")
    ap.add_argument("--static", type=int, nargs="*", default=[], help="static decode splits (both contexts)")
    ap.add_argument("--regroup", type=int, nargs="*", default=[],
                    help="adaptive_plan with front passes repartitioned every N layers (SURVEY §8(f) f4)")
    a = ap.parse_args()
    import torch
    from synth import Q7B, Q2B
    from synth.inputs import poisson_trace
    SHAPE = Q7B if a.model == "7b" else Q2B
    from paper_2509_21301_b200 import engine as E
    if a.offload:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from offload_bench import build as build_offload
        eng = build_offload(SHAPE, a.offload)
    else:
        eng = BN.build_engine(SHAPE, 0)
    curves, plan = BN.profile_and_plan(eng, False, lambda *x: print(*x, file=sys.stderr, flush=True))
    sv, sp = plan["best"][0], plan["best"][1]
    print(json.dumps({"plan": {"best": plan["best"][:2], "sm_min": plan["sm_min"]},
                      "t_d_dv_ms": [round(x, 2) for x in curves["t_d_dv_ms"]],
                      "t_v_ms": [round(x, 2) for x in curves["t_v_ms"]]}), flush=True)
    t_front = (0.5 * (curves["t_v_solo_ms"] + curves["t_v_solo_7920_ms"]) + curves["t_p_solo_ms"]) / 1000.0
    t_front_p = (curves["t_v_solo_ms"] + curves["t_p_solo_ms"]) / 1000.0   # cfg 2: 52x94 screenshots only
    pols = [("adaptive_plan", dict(mode=E.ADAPTIVE, sm_op_dv=sv, sm_op_dp=sp, sm_min=plan["sm_min"],
                                   alpha_dv=plan["alpha_dv"], alpha_dp=plan["alpha_dp"], b_max=16))]
    for op in a.sm_op:
        smin = min(plan["sm_min"], op)
        pols.append((f"adaptive_op{op}", dict(mode=E.ADAPTIVE, sm_op_dv=op, sm_op_dp=op, sm_min=smin,
                                              alpha_dv=(op - smin) / 3.0, alpha_dp=(op - smin) / 3.0, b_max=16)))
    for st in a.static:
        pols.append((f"static_{st}", dict(mode=E.STATIC, sm_decode_dv=st, sm_decode_dp=st, b_max=16)))
    for fl in a.floor:
        pols.append((f"adaptive_floor{fl}", dict(mode=E.ADAPTIVE, sm_op_dv=sv, sm_op_dp=sp, sm_min=plan["sm_min"],
                                                 alpha_dv=plan["alpha_dv"], alpha_dp=plan["alpha_dp"], b_max=16,
                                                 sm_dv_floor=fl)))
    for smin in a.sm_min:
        if smin > min(sv, sp):
            continue
        pols.append((f"adaptive_smin{smin}", dict(mode=E.ADAPTIVE, sm_op_dv=sv, sm_op_dp=sp, sm_min=smin,
                                                  alpha_dv=(sv - smin) / 3.0, alpha_dp=(sp - smin) / 3.0, b_max=16)))
    pols += [(f"adaptive_regroup{n}", dict(pols[0][1], front_regroup=n)) for n in a.regroup]
    base = {"serial": dict(mode=E.SERIAL, b_max=16), "multi_stream": dict(mode=E.MULTI_STREAM, b_max=16),
            "chunk_128": dict(mode=E.CHUNK, chunk_budget=128, b_max=16),
            "pf_limit_5": dict(mode=E.PF_LIMIT, pf_threshold=5, b_max=16)}
    pols += [(n, base[n]) for n in a.policies.split(",") if n in base]
    for rho in a.rho:
        trs = [(BN.make_trace(SHAPE, a.requests, rho, t_front, 61 + k) if a.trace == 'mmpp' else poisson_trace(a.requests, rho / t_front_p, 21 + k)) for k in range(a.seeds)]
        for name, pol in pols:
            eng.set_partition(**pol)
            rs = []
            t_pol = time.time()
            sw0 = eng.lib.nova_front_switches(eng.h)
            for k, tr in enumerate(trs):
                inputs = BN.make_inputs(SHAPE, tr, 400 + k, 0, True)
                r = BN.replay(eng, inputs)
                rs.append({"max": max(r["lat_ms"]), "p99": BN.pct(r["lat_ms"], 0.99),
                           "mean": statistics.mean(r["lat_ms"]), "rps": r["n"] / r["wall_s"]})
            print(json.dumps({"rho": rho, "policy": name,
                              **{k: round(statistics.mean(x[k] for x in rs), 2) for k in rs[0]},
                              "per_seed_max": [round(x["max"], 1) for x in rs],
                              "front_switches": eng.lib.nova_front_switches(eng.h) - sw0,
                              "wall_s": round(time.time() - t_pol, 1)}), flush=True)
    eng.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
