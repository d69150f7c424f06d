"""Layer-wise ViT weight offload on B200 (BASELINE configs[3];
mirrors PAPER.md Table layer_vision): single vision-forward latency and HBM
footprint with K = 2..5 physical layer slots vs all layers resident, the measured pinned
H2D bandwidth, and the Eq. 8 zero-stall bound B >= (S/T)(L-K)/(L-2).

    python scripts/offload_bench.py [--model 7b] [--iters 5]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(shape, K, device=0, serving=True):
    from synth.models import weight_specs
    from synth.weights import device_tensor
    from paper_2509_21301_b200 import engine as E
    if serving:   # the bench's serving limits (scripts/policy_sweep.py --offload)
        opts = E.EngineOptions(device=device, max_requests=64, max_decode_batch=16, kv_pages=2600, max_patches=7920,
                               max_prompt=128, max_gen=64, vit_resident_layers=K, use_green_ctx=1)
    else:
        opts = E.EngineOptions(device=device, max_requests=4, max_decode_batch=4, kv_pages=256, max_patches=7920,
                               max_prompt=128, max_gen=64, vit_resident_layers=K)
    eng = E.Engine(shape, opts)
    for name, shp, init in weight_specs(shape):
        if K > 0 and name.startswith("model.visual.blocks."):
            t = device_tensor(name, shp, init, 2, device=f"cuda:{device}").cpu()   # host source for the arena
        else:
            t = device_tensor(name, shp, init, 2, device=f"cuda:{device}")
        eng.load_tensor(name, t)
    torch.cuda.synchronize()
    eng.finalize()
    return eng


def h2d_bandwidth(nbytes=256 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from synth import Q7B, Q2B
    from synth.models import vit_layer_names, weight_specs
    from paper_2509_21301_b200.engine import nova_required_bandwidth
    shape = Q7B if a.model == "7b" else Q2B
    layer_bytes = sum(2 * int(torch.tensor(shp).prod()) for n, shp, _ in weight_specs(shape)
                      if n.startswith("model.visual.blocks.0."))
    L = shape.vit_depth
    bw = h2d_bandwidth()
    rows = []
    aware = None
    for K in (0, 2, 3, 4, 5):
        eng = build(shape, K, serving=False)
        res = {"K": K if K else "all", "weights_bytes": eng.memory["weights"],
               "vit_resident_bytes": (K if K else L) * layer_bytes}
        for grid in ((52, 94), (66, 120)):
            eng.time_pass(0, 0, *grid, iters=1)
            t = eng.time_pass(0, 0, *grid, iters=a.iters)[0]
            res[f"t_vision_ms_{grid[0]}x{grid[1]}"] = round(t, 3)
            if K:
                res[f"eq8_required_GBps_{grid[0]}x{grid[1]}"] = round(
                    nova_required_bandwidth(L * layer_bytes, t / 1e3, L, K) / 1e9, 1)
        rows.append(res)
        if K == 2:   # offload-aware split: vision pass vs decode split, co-running decode
            from paper_2509_21301_b200.engine import nova_offload_floor
            splits = [8 * k for k in range(1, 15)]
            tv = [eng.time_pass(0, sp, 52, 94, B=2, ctx=1334, corun=1, iters=2)[0] for sp in splits]
            t_h2d = L * layer_bytes / (bw * 1e9) * 1e3
            aware = {"K": 2, "t_h2d_ms": round(t_h2d, 2), "splits": splits, "t_v_ms": [round(x, 2) for x in tv],
                     "sm_dv_floor": nova_offload_floor(splits, tv, t_h2d)}
        eng.close()
        del eng
        torch.cuda.empty_cache()
    base = rows[0]
    for r in rows[1:]:
        for g in ("52x94", "66x120"):
            r[f"stall_ms_{g}"] = round(r[f"t_vision_ms_{g}"] - base[f"t_vision_ms_{g}"], 3)
    out = {"model": shape.name, "vit_layer_bytes": layer_bytes, "vit_layers": L, "pinned_h2d_GBps": round(bw, 1),
           "streamed_bytes_per_pass": L * layer_bytes, "rows": rows, "offload_aware_split": aware}
    print(json.dumps(out))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
