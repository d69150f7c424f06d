#!/usr/bin/env python
"""Nova on B200 -- serving benchmark (BASELINE.json metric: max & p99 request latency
(ms) at requests/sec; per-stage HBM / tensor-pipe % of peak).

A "step" is one replay, in real time, of a synthetic bursty GUI-agent trace
segment (R requests, MMPP-2 arrivals at utilisation rho; SURVEY.md §8(d) d1') through
the whole hot path: intake -> Algorithm 1 scheduler -> Eq. 5 adaptive split ->
green-context partitions -> vision encode / prefill / decode kernels -> token
emission (all rows of SURVEY §8(a)).  Workload = BASELINE configs[2]
(Qwen2-VL-7B-shaped, random init, 1080p screenshots, 32-128 prompt tokens,
32-64 output tokens).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

`value` = max E2E request latency (ms) over the timed steps with the screenshots
already resident in HBM; `e2e` = the same through host (pinned) buffers, H2D
inside the timed region.  N > 1 (torchrun): independent replicas, each replaying
its own trace (weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max & p99 request latency (ms) at requests/sec; per-stage HBM/tensor-pipe % peak"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="nova", choices=["nova", "reference"])
    p.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3"],
                   help="cfg2 = BASELINE configs[1] (2B, steady Poisson stream, static split sweep vs serial; "
                        "the default, as the metric is quoted on configs[1]); cfg3 = configs[2] (7B, bursty "
                        "MMPP-2 GUI-agent trace)")
    p.add_argument("--model", default=None, choices=["7b", "2b"], help="override the workload's model")
    p.add_argument("--no-solo-7b", action="store_true", help="cfg2: skip the 7B (cfg 3 shape) solo stage passes")
    p.add_argument("--rho", type=float, default=0.7)
    p.add_argument("--requests", type=int, default=None,
                   help="requests per step (per GPU); default cfg2: 96 (~2.4 s of Poisson arrivals), cfg3: 48")
    p.add_argument("--no-compare", action="store_true", help="skip the serial / static-50/50 comparison replays")
    p.add_argument("--compare-rho", type=float, nargs="*", default=None,
                   help="offered loads of the comparison (default cfg2: 0.7 0.9, cfg3: 0.5 0.7)")
    p.add_argument("--compare-seeds", type=int, default=3, help="traces per offered load in the comparison")
    p.add_argument("--quick", action="store_true", help="smaller profile sweep (debug)")
    p.add_argument("--skip-profile", action="store_true", help="no co-run curve sweep (ncu launch-list runs)")
    p.add_argument("--dispatch", default="jsq", choices=["jsq", "rr"], help="replica dispatcher policy (N > 1)")
    p.add_argument("--out", default=None, help="also write the JSON line here")
    return p.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- model + engine
def build_engine(shape, device, seed=2):
    import torch
    from synth.models import weight_specs
    from synth.weights import device_tensor
    from paper_2509_21301_b200 import engine as E
    # NOVA_BENCH_GREEN=0: partitions as SM-budget-limited grids on primary-context streams, for ncu launch
    # lists only (ncu does not profile kernels launched into green contexts); never for a bench number
    green = int(os.environ.get("NOVA_BENCH_GREEN", "1"))
    opts = E.EngineOptions(device=device, max_requests=64, max_decode_batch=16, kv_pages=2600, max_patches=7920,
                           max_prompt=128, max_gen=64, use_green_ctx=green)
    eng = E.Engine(shape, opts)
    for name, shp, init in weight_specs(shape):
        t = device_tensor(name, shp, init, seed, device=f"cuda:{device}")
        eng.load_tensor(name, t)
        del t
    torch.cuda.synchronize()
    eng.finalize()
    return eng


def profile_and_plan(eng, quick=False, log=print):
    """Measured latency-vs-SM curves (co-run) -> Eq. 1-3 planner -> Eq. 5 parameters."""
    from paper_2509_21301_b200 import engine as E
    total, g, nsplit = eng.query_sms()
    splits = [g * k for k in range(1, nsplit + 1)]
    if quick:
        splits = splits[::3]
    B_ref, ctx = 2, 1334
    # solo decode first (a cold GPU, as in a solo pass), then again after the tensor-heavy front passes
    # have pushed the part into its power-capped clock state (the serving regime): both are reported
    eng.time_pass(2, 0, B=B_ref, ctx=ctx, iters=3)               # warm the decode path first
    td_full = eng.time_pass(2, 0, B=B_ref, ctx=ctx, iters=10)[0]
    tv_solo = eng.time_pass(0, 0, 52, 94, iters=2)[0]
    tv_solo_b = eng.time_pass(0, 0, 66, 120, iters=2)[0]
    tp_solo = eng.time_pass(1, 0, 52, 94, 64, iters=2)[0]
    td_hot = eng.time_pass(2, 0, B=B_ref, ctx=ctx, iters=10)[0]
    tv, tp, tdv, tdp = [], [], [], []
    for s in splits:
        f, d = eng.time_pass(0, s, 52, 94, B=B_ref, ctx=ctx, corun=1, iters=2)
        tv.append(f)
        tdv.append(d)
        f, d = eng.time_pass(1, s, 52, 94, 64, B=B_ref, ctx=ctx, corun=1, iters=2)
        tp.append(f)
        tdp.append(d)
    # SM_min: TBT bound at the paper's ratio, 80 ms over its 28.9 ms solo decode iteration (
    # DESIGN.md R12)
    plan = E.nova_plan(splits, tv, tp, tdv, tdp, gen_len=48, tau=80.0 / 28.9, t_d_full=td_full)
    curves = {"splits": splits, "t_v_ms": tv, "t_p_ms": tp, "t_d_dv_ms": tdv, "t_d_dp_ms": tdp,
              "t_v_solo_ms": tv_solo, "t_v_solo_7920_ms": tv_solo_b, "t_p_solo_ms": tp_solo, "t_d_full_ms": td_full,
              "t_d_full_after_front_ms": td_hot,
              "B_ref": B_ref, "ctx_ref": ctx}
    log(f"[bench] curves solo: t_v {tv_solo:.2f}/{tv_solo_b:.2f} ms t_p {tp_solo:.2f} ms t_d {td_full:.3f} ms; "
        f"plan best {plan['best']} sm_min {plan['sm_min']}")
    return curves, plan


def make_trace(shape, n, rho, t_front_s, seed, kind="mmpp"):
    """cfg 3: MMPP-2 bursty GUI-agent mix at rho = lambda x T_front; cfg 2: Poisson arrivals at
    lambda = rho / T_front with fixed 52x94 screenshots, prompt 64, gen_len 48 (SURVEY.md §8(d) d1')."""
    from synth.inputs import mmpp2_trace, poisson_trace
    if kind == "poisson":
        return poisson_trace(n, rho / t_front_s, seed)
    return mmpp2_trace(n, rho, t_front_s, seed)


def solo_stage_fracs(shape, tv_ms, tp_ms, td_ms, td_hot_ms, hbm, tfl, B_ref=2, ctx=1334):
    """Solo stage passes on the full GPU against the measured peaks: algorithmic FLOPs / bytes of
    SURVEY.md §8(d) d2 (N = 4888 patches, S = 1222 + 64 tokens, decode B_ref at ctx) over the time."""
    D, F, V = shape.llm_dim, shape.llm_ffn, shape.vocab
    N = 52 * 94
    fl_v = 32 * (2 * N * (1280 * 3840 + 1280 ** 2 + 2 * 1280 * 5120) + 4 * N * N * 1280) + \
        2 * N * 1176 * 1280 + 2 * (N // 4) * (5120 ** 2 + 5120 * D)
    S, H, KV, hd = 1222 + 64, shape.llm_heads, shape.llm_kv_heads, shape.head_dim
    fl_p = shape.llm_layers * (2 * S * (D * (D + 2 * KV * hd) + D * D + 3 * D * F) + 2 * S * S * H * hd) + 2 * D * V
    out = {}
    for name, fl, ms in (("vision_encode_N4888", fl_v, tv_ms), ("prefill_S1286", fl_p, tp_ms)):
        if ms:
            ach = fl / (ms / 1e3) / 1e12
            out[name] = {"ms": round(ms, 3), "achieved": round(ach, 1), "unit": "TFLOP/s", "peak": tfl,
                         "frac": round(ach / tfl, 4), "bound": "tensor"}
    Wb = shape.llm_layers * 2 * (D * (D + 2 * KV * hd) + D * D + 3 * D * F) + 2 * D * V   # bf16 bytes
    kvb = B_ref * (ctx + 1) * shape.llm_layers * 2 * KV * hd * 2
    for tag, ms in (("", td_ms), ("_after_front_passes", td_hot_ms)):
        if ms:
            ach = (Wb + kvb) / (ms / 1e3) / 1e9
            out[f"decode_B{B_ref}_ctx{ctx}{tag}"] = {"ms": round(ms, 3), "achieved": round(ach, 1), "unit": "GB/s",
                                                     "peak": hbm, "frac": round(ach / hbm, 4), "bound": "hbm"}
    return out


def make_inputs(shape, rows, seed, device, resident):
    """Pixels + prompt ids per request; resident=True -> pixels pre-staged in HBM."""
    import numpy as np
    import torch
    from synth.inputs import make_request
    out = []
    cache = {}
    for i, r in enumerate(rows):
        key = (r.grid_h, r.grid_w)
        if key not in cache:      # screenshot content does not affect timing; one image per size
            cache[key] = make_request(shape, key, 1, 1, seed + len(cache)).pixels
        pix = cache[key]
        rng = np.random.default_rng(seed * 1000 + i)
        ids = rng.integers(0, shape.vocab, r.prompt_tokens).astype(np.int32)
        t = torch.from_numpy(pix.view(np.int16))
        t = t.cuda(device) if resident else t.pin_memory()
        out.append((t, ids, r.gen_len, r.arrival_s))
    return out


def replay(eng, inputs, t0=None, rank=0, world=1, board=None, policy="jsq"):
    """Submit at the trace's arrival times (real time), step the scheduler until every request
    finished.  With world > 1 the trace is global: rank 0's dispatcher assigns each arrival to a
    replica (JSQ on the published front backlog) and each rank submits only its own requests.
    Returns per-request latencies, the step wall time and host<->device bytes."""
    import ctypes as C
    from paper_2509_21301_b200 import _abi as A
    from paper_2509_21301_b200.dispatch import Dispatcher, wait_assignment
    n = len(inputs)
    ids = {}
    if t0 is None:
        t0 = time.monotonic_ns() + 2_000_000   # first arrival 2 ms from now
    base_finished = eng.step(0).finished
    h2d = 0
    sub_err = []
    state = {"submitted": 0, "done": False}

    def submitter():
        nonlocal h2d
        try:
            for i, (pix, prm, gen, at) in enumerate(inputs):
                target = t0 + int(at * 1e9)
                while True:
                    dt = target - time.monotonic_ns()
                    if dt <= 0:
                        break
                    time.sleep(min(dt / 1e9, 0.002))
                if world > 1 and wait_assignment(board, i) != rank:
                    continue
                r = A.Request()
                r.pixels_bf16 = pix.data_ptr()
                r.height, r.width = int(pix.shape[1]), int(pix.shape[2])
                r.prompt_ids = prm.ctypes.data
                r.n_prompt = len(prm)
                r.gen_len = gen
                r.arrival_ns = target
                rid = A.U64()
                while True:
                    rc = eng.lib.nova_submit(eng.h, C.byref(r), C.byref(rid))
                    if rc != -4:
                        break
                    time.sleep(0.0005)
                if rc != 0:
                    raise RuntimeError(f"submit failed {rc}")
                ids[rid.value] = i
                state["submitted"] += 1
                if not pix.is_cuda:
                    h2d += pix.numel() * 2
                h2d += len(prm) * 4
        except Exception as ex:  # pragma: no cover
            sub_err.append(ex)
        state["done"] = True

    def dispatcher():
        d = Dispatcher(board, [x[3] for x in inputs], policy)
        while not d.done():
            d.assign_due((time.monotonic_ns() - t0) / 1e9)
            time.sleep(0.0001)

    threads = [threading.Thread(target=submitter)]
    if world > 1 and rank == 0:
        threads.append(threading.Thread(target=dispatcher))
    for th in threads:
        th.start()
    toks, first = [], 0
    last_progress = time.monotonic()
    while True:
        info = eng.step(500)
        if sub_err:
            raise sub_err[0]
        new = eng.poll_tokens(1 << 16)
        if new or info.events:
            last_progress = time.monotonic()
        elif time.monotonic() - last_progress > 120.0:   # watchdog: report a stall instead of hanging
            log = eng.decision_log()
            raise RuntimeError(f"replay stalled 120 s: submitted {state['submitted']}, finished "
                               f"{info.finished - base_finished}, pending {info.n_pending}, active {info.active}, "
                               f"last decisions {log[-6:]}")
        toks += new
        first += sum(1 for t in new if t[1] == 0)
        if board is not None:
            board.publish(rank, state["submitted"] - first, state["submitted"])
        if state["done"] and info.finished - base_finished >= state["submitted"]:
            break
    for th in threads:
        th.join()
    t1 = time.monotonic_ns()
    toks += eng.poll_tokens(1 << 20)
    lat, ttft, qwait, front = [], [], [], []
    for rid in ids:
        st = eng.stats(rid)
        lat.append((st["last_tok"] - st["arrival"]) / 1e6)
        ttft.append((st["first_tok"] - st["arrival"]) / 1e6)
        qwait.append(max(0, st["vis_start"] - st["arrival"]) / 1e9)
        front.append((st["pre_end"] - st["vis_start"]) / 1e9)
    d2h = 4 * len(toks)
    first_arrival = t0 + int(inputs[0][3] * 1e9)
    return {"lat_ms": lat or [0.0], "ttft_ms": ttft or [0.0], "wall_s": (t1 - first_arrival) / 1e9, "h2d": h2d,
            "d2h": d2h, "tokens": len(toks), "n": len(ids), "qwait_s": qwait, "front_s": front,
            "span_s": (inputs[-1][3] - inputs[0][3])}


def pct(xs, q):
    s = sorted(xs)
    k = max(0, math.ceil(q * len(s)) - 1)
    return s[k]


# ---------------------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_sample(shape, reps=1):
    """Bounded sample of the same workload on the host: one full-width ViT layer (N=4888), one
    prefill LLM layer (S=1286) and one decode LLM layer (ctx 1334) of the oracle, timed, then
    extrapolated to one request (32 ViT + 28 prefill + 47 x 28 decode layers)."""
    import numpy as np
    from oracle import vlm as V
    from synth.models import reduced_depth
    from synth.weights import gen_tensor
    from synth.models import weight_specs
    s1 = reduced_depth(shape, 1, 1)
    specs = {n: (shp, init) for n, shp, init in weight_specs(s1)}
    need = [n for n in specs if n.startswith("model.visual.blocks.0.") or n.startswith("model.language_model.layers.0.")]
    W = V.OracleWeights({n: gen_tensor(n, specs[n][0], specs[n][1], 2) for n in need}, np.float32)
    rng = np.random.default_rng(0)
    N, S, ctx = 4888, 1286, 1334
    x = rng.standard_normal((N, shape.vit_dim)).astype(np.float32)
    hp, wp = np.divmod(np.arange(N), 94)
    cos, sin = V.vit_rope_tables(hp, wp, shape.vit_head_dim, shape.vit_theta, np.float32)
    xl = rng.standard_normal((S, shape.llm_dim)).astype(np.float32)
    pos = V.mrope_positions(52, 94, S - 1222, 2)
    c2, s2 = V.mrope_tables(pos, shape.head_dim, shape.llm_theta, shape.mrope_section, np.float32)
    times = {"vit_layer": [], "prefill_layer": [], "decode_layer": []}
    for _ in range(reps):
        t = time.perf_counter()
        V.vit_block(x, W, 0, s1, cos, sin)
        times["vit_layer"].append(time.perf_counter() - t)
        cache = {"k": {}, "v": {}}
        t = time.perf_counter()
        V.llm_layer(xl, W, 0, s1, c2, s2, cache, 0)
        times["prefill_layer"].append(time.perf_counter() - t)
        xd = xl[:1]
        pd = np.full((3, 1), ctx)
        cd, sd = V.mrope_tables(pd, shape.head_dim, shape.llm_theta, shape.mrope_section, np.float32)
        pad = ctx - S
        cache["k"][0] = np.concatenate([cache["k"][0], cache["k"][0][:pad]])
        cache["v"][0] = np.concatenate([cache["v"][0], cache["v"][0][:pad]])
        t = time.perf_counter()
        V.llm_layer(xd, W, 0, s1, cd, sd, cache, ctx)
        times["decode_layer"].append(time.perf_counter() - t)
    med = {k: statistics.median(v) for k, v in times.items()}
    per_req_s = shape.vit_depth * med["vit_layer"] + shape.llm_layers * med["prefill_layer"] + \
        47 * shape.llm_layers * med["decode_layer"]
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count()])
    except Exception:
        cores = os.cpu_count()
    return per_req_s * 1000.0, med, cores


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import Q7B, Q2B
    model = args.model or ("2b" if args.workload == "cfg2" else "7b")
    shape = Q7B if model == "7b" else Q2B
    for _ in range(args.warmup):
        cpu_oracle_sample(shape)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, med, cores = cpu_oracle_sample(shape)
        vals.append(v)
    el = time.perf_counter() - t0
    value = statistics.median(vals)
    sample = (f"oracle/vlm.py fp32 NumPy: 1 ViT layer (N=4888) + 1 prefill layer (S=1286) + 1 decode layer "
              f"(ctx 1334) at {shape.name} width, extrapolated to one request (32 + 28 + 47x28 layers); "
              f"medians {json.dumps({k: round(x, 3) for k, x in med.items()})} s")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el * 1000 / args.steps, 1),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": ("BASELINE configs[1]: 2B-shaped, Poisson stream (single-request "
                                                         "latency of the CPU oracle)" if args.workload == "cfg2" else
                                                         "BASELINE configs[2]: 7B-shaped bursty GUI-agent trace "
                                                         "(single-request latency of the CPU oracle)"),
                                            "model": shape.name},
            "cpu_baseline": {"value": round(value, 1), "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if args.out:
        open(args.out, "w").write(json.dumps(line) + "\n")
    return 0


# ---------------------------------------------------------------------------- main (nova)
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (functional check of the replica path on a one-GPU box): every rank on GPU 0, gloo
    if os.environ.get("NOVA_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("NOVA_BENCH_SAME_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if rank == 0 else (lambda *a: None)
    from synth import Q7B, Q2B
    from paper_2509_21301_b200 import engine as E
    model = args.model or ("2b" if args.workload == "cfg2" else "7b")
    shape = Q7B if model == "7b" else Q2B
    kind = "poisson" if args.workload == "cfg2" else "mmpp"
    if args.requests is None:
        args.requests = 96 if kind == "poisson" else 48
    compare_rho = args.compare_rho if args.compare_rho is not None else ([0.7, 0.9] if kind == "poisson" else [0.5, 0.7])
    pk = peaks()
    t_setup = time.time()
    eng = build_engine(shape, local)
    log(f"[bench] engine ready in {time.time() - t_setup:.1f}s; memory {eng.memory}")
    if args.skip_profile:   # ncu launch-list runs: no co-run sweep, fixed plan, solo curve points only
        tv = eng.time_pass(0, 0, 52, 94, iters=1)[0]
        curves = {"t_v_solo_ms": tv, "t_v_solo_7920_ms": 1.6 * tv, "t_p_solo_ms": eng.time_pass(1, 0, 52, 94, 64,
                                                                                               iters=1)[0]}
        plan = {"best": (88, 88, 0.0, 0.0), "sm_min": 32, "alpha_dv": 18.667, "alpha_dp": 18.667}
    else:
        curves, plan = profile_and_plan(eng, args.quick, log)
    sv, sp = plan["best"][0], plan["best"][1]
    if plan.get("points"):
        eng.set_frontier(plan["points"], window=16)   # FRONTIER mode
    policy = dict(mode=E.ADAPTIVE, sm_op_dv=sv, sm_op_dp=sp, sm_min=plan["sm_min"], alpha_dv=plan["alpha_dv"],
                  alpha_dp=plan["alpha_dp"], b_max=16)
    eng.set_partition(**policy)
    # T_front: request-mix mean of solo t_v + t_p (cfg 3: half 4888-patch, half 7920-patch screenshots;
    # cfg 2: 4888-patch screenshots, prompt 64)
    if kind == "poisson":
        t_front = (curves["t_v_solo_ms"] + curves["t_p_solo_ms"]) / 1000.0
    else:
        t_front = (0.5 * (curves["t_v_solo_ms"] + curves["t_v_solo_7920_ms"]) + curves["t_p_solo_ms"]) / 1000.0
    # global trace (identical on every rank): world x requests at world x the per-GPU load (weak scaling)
    traces = [make_trace(shape, args.requests * world, args.rho * world, t_front, 31 + i, kind)
              for i in range(args.warmup + 2 * args.steps + 2)]
    counter = [0]

    def run_step(tr, seed, resident):
        inputs = make_inputs(shape, tr, seed, local, resident)
        if world == 1:
            return replay(eng, inputs)
        from paper_2509_21301_b200.dispatch import ReplicaBoard
        counter[0] += 1
        name = f"nova_{os.environ.get('MASTER_PORT', '0')}_{counter[0]}"
        board = ReplicaBoard(name, world, len(inputs), create=True) if rank == 0 else None
        dist.barrier()
        if rank != 0:
            board = ReplicaBoard(name, world, len(inputs), create=False)
        t0 = torch.tensor([time.monotonic_ns() + 200_000_000], dtype=torch.int64, device="cuda")
        dist.broadcast(t0, 0)
        r = replay(eng, inputs, int(t0.item()), rank, world, board, args.dispatch)
        dist.barrier()
        board.close()
        return r

    # warm-up steps (untimed)
    for i in range(args.warmup):
        run_step(traces[i], 100 + i, True)
    eng.kernel_stats_reset()
    eng.kernel_timing(4)
    launches0 = eng.lib.nova_launch_count()
    log(f"[bench] libnova launches before the timed region: {launches0}")
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    prof_range = os.environ.get("NOVA_PROFILER_RANGE") == "1"   # ncu --profile-from-start off
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    res = []
    for i in range(args.steps):       # inputs resident in HBM
        res.append(run_step(traces[args.warmup + i], 200 + i, True))
    torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    launches = eng.lib.nova_launch_count() - launches0
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    ks = eng.kernel_stats()
    ks_sm = eng.kernel_stats_sm()
    eng.kernel_timing(0)
    # end-to-end: pinned host screenshots, H2D inside the timed region
    res_e2e = []
    for i in range(args.steps):
        res_e2e.append(run_step(traces[args.warmup + args.steps + i], 300 + i, False))
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)

    def agg(rs):
        lat = [x for r in rs for x in r["lat_ms"]]
        wall = sum(r["wall_s"] for r in rs)
        return {"max_ms": max(lat), "p99_ms": pct(lat, 0.99), "mean_ms": statistics.mean(lat),
                "ttft_p99_ms": pct([x for r in rs for x in r["ttft_ms"]], 0.99), "n": sum(r["n"] for r in rs),
                "wall_s": wall,
                "h2d": sum(r["h2d"] for r in rs) / len(rs), "d2h": sum(r["d2h"] for r in rs) / len(rs)}

    A, Ae = agg(res), agg(res_e2e)
    # Eq. 6: M/G/1 prediction of the vision-queue wait from the measured front service
    qw = [x for r in res for x in r["qwait_s"]]
    fs = [x for r in res for x in r["front_s"]]
    lam = sum(r["n"] for r in res) / max(1e-9, sum(r["span_s"] for r in res))
    ET, ET2 = statistics.mean(fs), statistics.mean([x * x for x in fs])
    rho_m = lam * ET
    mg1 = {"lambda_rps": round(lam, 3), "E_T_ms": round(ET * 1e3, 2), "E_T2_ms2": round(ET2 * 1e6, 1),
           "utilization": round(rho_m, 3), "measured_wait_ms": round(statistics.mean(qw) * 1e3, 2),
           "predicted_wait_ms": round(lam * ET2 / (2 * (1 - rho_m)) * 1e3, 2) if rho_m < 1 else None,
           "note": "bursty MMPP arrivals, so M/G/1 (Poisson) is expected to under-predict"}
    # Comparison (SURVEY.md §8(d) pass criteria): adaptive vs serial stage execution vs a static 50/50
    # split on the SAME traces, 3 seeds per offered load; "beats X" = lower mean-over-seeds max E2E and
    # lower in >= 2 of 3 seeds, at req/s >= 0.99 x X's.
    compare = {}
    if not args.no_compare:
        pols = [("adaptive", policy),
                ("static_50_50", dict(mode=E.STATIC, sm_decode_dv=72, sm_decode_dp=72, b_max=16)),
                ("serial", dict(mode=E.SERIAL, b_max=16)),
                # the paper's baselines: prefill-first with decode threshold 5, and
                # co-running stages with no SM partition (both streams see every SM)
                ("pf_limit_5", dict(mode=E.PF_LIMIT, pf_threshold=5, b_max=16)),
                ("multi_stream", dict(mode=E.MULTI_STREAM, b_max=16)),
                # the paper's chunked-prefill baseline: hybrid prefill-chunk + decode batches,
                # token budget 128 (the paper's best)
                ("chunk_128", dict(mode=E.CHUNK, chunk_budget=128, b_max=16)),
                # the same adaptive policy, front passes repartitioned every 8 layers
                ("adaptive_regroup8", dict(policy, front_regroup=8))]
        if plan.get("points"):   # Pareto point for the estimated arrival rate
            pols.append(("frontier", dict(mode=E.FRONTIER, b_max=16)))
        if kind == "poisson":    # cfg 2: the static SM-split sweep
            pols += [(f"static_{s_}", dict(mode=E.STATIC, sm_decode_dv=s_, sm_decode_dp=s_, b_max=16))
                     for s_ in (24, 48, 96)]
        for rho in compare_rho:
            trs = [make_trace(shape, args.requests, rho, t_front, 61 + k, kind) for k in range(args.compare_seeds)]
            runs = {name: [] for name, _ in pols}
            for k, tr in enumerate(trs):
                for name, pol in pols:
                    eng.set_partition(**pol)
                    r = agg([run_step(tr, 400 + k, True)])
                    runs[name].append({"max_ms": round(r["max_ms"], 2), "p99_ms": round(r["p99_ms"], 2),
                                       "mean_ms": round(r["mean_ms"], 2),
                                       "req_per_s": round(r["n"] / r["wall_s"], 3)})
            summ = {}
            for name, rs in runs.items():
                summ[name] = {k: round(statistics.mean(x[k] for x in rs), 2) for k in rs[0]}
                summ[name]["per_seed_max_ms"] = [x["max_ms"] for x in rs]
            ad = runs["adaptive"]
            verdict = {}
            for name in [n for n, _ in pols if n != "adaptive"]:
                xs = runs[name]
                wins = sum(a["max_ms"] < b["max_ms"] for a, b in zip(ad, xs))
                verdict[name] = {"lower_mean_max": summ["adaptive"]["max_ms"] < summ[name]["max_ms"],
                                 "seeds_won": wins,
                                 "rps_ratio": round(summ["adaptive"]["req_per_s"] / summ[name]["req_per_s"], 3)}
                verdict[name]["beats"] = bool(verdict[name]["lower_mean_max"] and wins >= 2 and
                                              verdict[name]["rps_ratio"] >= 0.99)
            compare[f"rho_{rho}"] = {"policies": summ, "adaptive_vs": verdict, "seeds": args.compare_seeds}
        eng.set_partition(**policy)

    # replicas: latencies of every rank pooled (exact global max / p99), wall time = max over ranks
    loc = torch.tensor([A["wall_s"], Ae["wall_s"], dev_ms], dtype=torch.float64, device="cuda")
    lat_all = [x for r in res for x in r["lat_ms"]]
    lat_all_e = [x for r in res_e2e for x in r["lat_ms"]]
    if dist:
        dist.all_reduce(loc, op=dist.ReduceOp.MAX)
        g = [None] * world
        dist.all_gather_object(g, (lat_all, lat_all_e))
        lat_all = [x for a, _ in g for x in a]
        lat_all_e = [x for _, b in g for x in b]
    wall, wall_e, dev_ms = loc.tolist()
    mx, p99, n_all = max(lat_all), pct(lat_all, 0.99), len(lat_all)
    mx_e, p99_e, n_all_e = max(lat_all_e), pct(lat_all_e, 0.99), len(lat_all_e)

    # roofline of the dominant kernel (largest summed device time among kernel classes)
    hbm = pk["hbm_gbs"]
    tfl = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    kernels = {}
    for name, (ms, work, n) in ks.items():
        if n == 0 or ms <= 0:
            continue
        unit = E.KERNEL_UNITS[name]
        # SURVEY §8(d) d2 "partition-normalized": the same rate over the SM-share-weighted time (each
        # launch's ms x its pass's SM budget / 148), i.e. what the per-SM rate would give on the whole GPU
        sm_ms = ks_sm.get(name, 0.0)
        share = sm_ms / ms if sm_ms > 0 else None
        if unit == "bytes":
            ach = work / (ms / 1e3) / 1e9
            kernels[name] = {"ms_per_launch": ms / n, "launches_timed": n, "achieved": round(ach, 1),
                             "unit": "GB/s", "frac": round(ach / hbm, 4)}
            if share:
                kernels[name]["mean_sm_share"] = round(share, 3)
                kernels[name]["frac_partition_normalized"] = round(ach / share / hbm, 4)
        else:
            ach = work / (ms / 1e3) / 1e12
            kernels[name] = {"ms_per_launch": ms / n, "launches_timed": n, "achieved": round(ach, 1),
                             "unit": "TFLOP/s", "frac": round(ach / tfl, 4)}
            if share:
                kernels[name]["mean_sm_share"] = round(share, 3)
                kernels[name]["frac_partition_normalized"] = round(ach / share / tfl, 4)
    kern_only = {k: v for k, v in kernels.items() if not k.endswith("_pass")}
    dom = max(kern_only, key=lambda k: ks[k][0]) if kern_only else None
    traffic = None
    try:
        nc = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = nc.get(shape.name, {}).get(dom)   # per model (profiles/ncu_traffic.json)
    except Exception:
        pass
    roof = None
    if dom:
        d = kernels[dom]
        roof = {"kernel": dom, "bound": "hbm" if d["unit"] == "GB/s" else "tensor", "achieved": d["achieved"],
                "peak": hbm if d["unit"] == "GB/s" else tfl, "unit": d["unit"], "frac": d["frac"],
                "traffic": traffic,
                # timed inside the serving replay on the decode / front partition; the same over the
                # SM-share-weighted time, and the mean SM share of those launches
                "frac_partition_normalized": d.get("frac_partition_normalized"),
                "mean_sm_share": d.get("mean_sm_share"),
                "peak_source": "MEASURED_PEAKS.json" + (" (fallback)" if pk.get("_fallback") else "") +
                ("" if d["unit"] == "GB/s" else " bf16_tflops_sustained")}
    stages = {k: v for k, v in kernels.items() if k.endswith("_pass")}
    # Solo stage passes on the full GPU (the §8(d) bars apply here), timed with CUDA events in this
    # run by the curve profiler: algorithmic FLOPs / bytes of SURVEY.md §8(d) d2 over the pass time
    stages_solo = solo_stage_fracs(shape, curves.get("t_v_solo_ms"), curves.get("t_p_solo_ms"),
                                   curves.get("t_d_full_ms"), curves.get("t_d_full_after_front_ms"), hbm, tfl,
                                   curves.get("B_ref", 2), curves.get("ctx_ref", 1334)) if curves.get("t_v_solo_ms") else {}

    line = {"metric": METRIC, "value": round(mx, 2), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 1), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, "
            "seeded screenshots/prompts, " + ("Poisson arrivals)" if kind == "poisson" else "MMPP-2 bursty arrivals)"),
            "p99_ms": round(p99, 2), "req_per_s": round(n_all / wall, 3),
            "config": {"workload": ("BASELINE configs[1]: Qwen2-VL-2B-shaped random init, steady Poisson request "
                                    "stream, static SM-split sweep vs serial execution" if kind == "poisson" else
                                    "BASELINE configs[2]: Qwen2-VL-7B-shaped random init, bursty synthetic "
                                    "GUI-agent trace, adaptive Pareto repartitioning"),
                       "model": shape.name, "requests_per_step_per_gpu": args.requests, "rho": args.rho,
                       "t_front_ms": round(t_front * 1000, 2),
                       "images": ("52x94 (4888 patches)" if kind == "poisson" else
                                  "50% 52x94 (4888 patches) / 50% 66x120 (7920 patches)"),
                       "prompt": "64" if kind == "poisson" else "U{32..128}",
                       "gen_len": "48" if kind == "poisson" else "U{32..64}",
                       "policy": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in policy.items()},
                       "l2": f"weights {eng.memory['weights'] / 1e9:.1f} GB streamed per pass >> 126 MB L2 "
                             "(no flush needed)", "parallelism": f"replicas x{world} ({args.dispatch} dispatcher)"},
            "e2e": {"value": round(mx_e, 2), "unit": "ms", "p99_ms": round(p99_e, 2),
                    "req_per_s": round(n_all_e / wall_e, 3), "h2d_bytes_per_step": int(Ae["h2d"]),
                    "d2h_bytes_per_step": int(Ae["d2h"])},
            "gpu_launches": int(launches), "roofline": roof, "stages_solo": stages_solo, "stages": stages,
            "kernels": kernels,
            "curves": {k: ([round(x, 3) for x in v] if isinstance(v, list) else (round(v, 3) if isinstance(v, float)
                                                                                else v)) for k, v in curves.items()},
            "plan": {"best": plan["best"][:2], "e2e_ms": round(plan["best"][2], 2), "thr_rps": round(plan["best"][3], 2),
                     "sm_min": plan["sm_min"], "alpha_dv": round(plan["alpha_dv"], 3),
                     "alpha_dp": round(plan["alpha_dp"], 3)},
            "compare": compare, "mg1": mg1, "clocks": clk}
    if os.environ.get("NOVA_BENCH_GREEN", "1") == "0":
        line["config"]["partitions"] = "NOT green contexts (NOVA_BENCH_GREEN=0, ncu launch-list run): not a bench number"
    if kind == "poisson" and not args.no_solo_7b and world == 1:
        # the §8(d) stage bars are stated at the cfg 3 (7B) shapes: time those solo passes too
        try:
            eng.close()
            eng = None
            eng7 = build_engine(Q7B, local)
            eng7.time_pass(2, 0, B=2, ctx=1334, iters=3)
            td7 = eng7.time_pass(2, 0, B=2, ctx=1334, iters=10)[0]
            eng7.time_pass(0, 0, 52, 94, iters=1)
            tv7 = eng7.time_pass(0, 0, 52, 94, iters=2)[0]
            tp7 = eng7.time_pass(1, 0, 52, 94, 64, iters=2)[0]
            td7h = eng7.time_pass(2, 0, B=2, ctx=1334, iters=10)[0]
            line["stages_solo_cfg3_7b"] = solo_stage_fracs(Q7B, tv7, tp7, td7, td7h, hbm, tfl)
            eng7.close()
        except Exception as ex:  # pragma: no cover
            line["stages_solo_cfg3_7b"] = {"error": str(ex)}
    if rank == 0 and world == 1:
        try:
            v, med, cores = cpu_oracle_sample(shape)
            line["cpu_baseline"] = {"value": round(v, 1), "unit": "ms", "cores": cores, "kind": "oracle",
                                    "sample": "oracle/vlm.py fp32 NumPy: 1 ViT layer (N=4888) + 1 prefill layer "
                                              "(S=1286) + 1 decode layer (ctx 1334), extrapolated to one request "
                                              f"latency; medians {json.dumps({k: round(x, 3) for k, x in med.items()})} s"}
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            open(args.out, "w").write(json.dumps(line) + "\n")
    if eng is not None:
        eng.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    try:
        rc = main()
    except Exception as ex:   # report and exit without joining possibly stuck engine threads
        import traceback
        traceback.print_exc()
        print(json.dumps({"metric": METRIC, "error": f"{type(ex).__name__}: {ex}"[:2000]}), flush=True)
        sys.stderr.flush()
        os._exit(1)
    sys.exit(rc)
