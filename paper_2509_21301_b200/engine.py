"""Python binding of include/nova.h -- argument marshalling only.

Every step of the path (encode, prefill, decode, scheduling, partitioning,
offload) runs inside libnova.so; torch provides the device buffers.  Module
functions carry the C names (nova_plan, nova_adaptive_sm, ...); `Engine` wraps an
opaque nova_engine* and calls nova_create / nova_submit / nova_step / ...
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi as A
from ._lib import lib

SERIAL, STATIC, ADAPTIVE, PF_LIMIT, MULTI_STREAM, FRONTIER, CHUNK = 0, 1, 2, 3, 4, 5, 6
CTX_DV, CTX_DP, CTX_SOLO = 0, 1, 2
DEC_VISION, DEC_PREFILL, DEC_DECODE, DEC_FINISH = 0, 1, 2, 3
EV_VISION_DONE, EV_PREFILL_DONE, EV_DECODE_DONE, EV_ARRIVAL = 0, 1, 2, 3
BACKEND_GPU, BACKEND_SIM = 0, 1
# NOVA_K_* classes (nova.h) and the unit of their algorithmic work
KERNEL_CLASSES = ["dec_gemv", "vit_gemm", "llm_gemm", "vit_attn", "pre_attn", "dec_attn", "lm_head", "vit_pass",
                  "pre_pass", "dec_pass", "dec_fused"]
KERNEL_UNITS = {"dec_gemv": "bytes", "vit_gemm": "flops", "llm_gemm": "flops", "vit_attn": "flops",
                "pre_attn": "flops", "dec_attn": "bytes", "lm_head": "bytes", "vit_pass": "flops",
                "pre_pass": "flops", "dec_pass": "bytes", "dec_fused": "bytes"}


class NovaError(RuntimeError):
    pass


def model_config(shape) -> A.ModelConfig:
    mc = A.ModelConfig()
    for f in ("vit_depth", "vit_dim", "vit_heads", "vit_mlp", "patch", "temporal_patch", "merge", "in_ch",
              "llm_layers", "llm_dim", "llm_heads", "llm_kv_heads", "head_dim", "llm_ffn", "vocab"):
        setattr(mc, f, int(getattr(shape, f)))
    mc.tie_embed = int(bool(shape.tie_embed))
    mc.mrope_section = (A.I32 * 3)(*shape.mrope_section)
    mc.vit_theta, mc.llm_theta = shape.vit_theta, shape.llm_theta
    mc.ln_eps, mc.rms_eps = shape.ln_eps, shape.rms_eps
    return mc


@dataclass
class EngineOptions:
    backend: int = BACKEND_GPU
    device: int = 0
    max_requests: int = 32
    max_decode_batch: int = 16
    kv_pages: int = 1024
    max_patches: int = 7920
    max_prompt: int = 128
    max_gen: int = 64
    vit_resident_layers: int = 0
    use_green_ctx: int = 1
    debug_keep_logits: int = 0
    finished_retention: int = 0   # 0: the engine default (4096 finished requests), < 0: keep all

    def cstruct(self) -> A.EngineConfig:
        ec = A.EngineConfig()
        for f in ("backend", "device", "max_requests", "max_decode_batch", "kv_pages", "max_patches", "max_prompt",
                  "max_gen", "vit_resident_layers", "use_green_ctx", "debug_keep_logits", "finished_retention"):
            setattr(ec, f, int(getattr(self, f)))
        return ec


def nova_query_memory(shape, opts: EngineOptions) -> dict:
    w, k, ws, ph = A.U64(), A.U64(), A.U64(), A.U64()
    mc, ec = model_config(shape), opts.cstruct()
    rc = lib().nova_query_memory(C.byref(mc), C.byref(ec), C.byref(w), C.byref(k), C.byref(ws), C.byref(ph))
    if rc != 0:
        raise NovaError(f"nova_query_memory -> {rc}")
    return {"weights": w.value, "kv": k.value, "workspace": ws.value, "pinned_host": ph.value}


class Engine:
    def __init__(self, shape, opts: EngineOptions | None = None):
        self.shape = shape
        self.opts = opts or EngineOptions()
        self.lib = lib()
        self._mc = model_config(shape)
        self._ec = self.opts.cstruct()
        self._keep = []
        bufs = None
        if self.opts.backend == BACKEND_GPU:
            import torch
            mem = nova_query_memory(shape, self.opts)
            dev = torch.device("cuda", self.opts.device)
            self._w = torch.empty(mem["weights"], dtype=torch.uint8, device=dev)
            self._kv = torch.empty(mem["kv"], dtype=torch.uint8, device=dev)
            self._ws = torch.empty(mem["workspace"], dtype=torch.uint8, device=dev)
            bufs = A.Buffers(self._w.data_ptr(), mem["weights"], self._kv.data_ptr(), mem["kv"],
                             self._ws.data_ptr(), mem["workspace"])
            self.memory = mem
        self.h = A.P()
        rc = self.lib.nova_create(C.byref(self._mc), C.byref(self._ec), C.byref(bufs) if bufs else None,
                                  C.byref(self.h))
        if rc != 0:
            raise NovaError(f"nova_create -> {rc}: {self.lib.nova_last_error(None)}")

    # -------------------------------------------------------------- helpers
    def _check(self, rc, what):
        if rc != 0:
            msg = self.lib.nova_last_error(self.h)
            raise NovaError(f"{what} -> {rc}: {msg.decode() if msg else ''}")

    def close(self):
        if self.h:
            self.lib.nova_destroy(self.h)
            self.h = A.P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- setup
    def load_tensor(self, name: str, t) -> None:
        """t: numpy uint16 bf16 bits (host) or a torch bf16/int16 tensor (host or device)."""
        if isinstance(t, np.ndarray):
            a = np.ascontiguousarray(t)
            assert a.dtype == np.uint16
            self._check(self.lib.nova_load_tensor(self.h, name.encode(), a.ctypes.data, a.nbytes, 0), name)
        else:
            t = t.contiguous()
            self._check(self.lib.nova_load_tensor(self.h, name.encode(), t.data_ptr(), t.numel() * t.element_size(),
                                                  int(t.is_cuda)), name)

    def load_weights(self, tensors: dict) -> None:
        for n, t in tensors.items():
            self.load_tensor(n, t)

    def finalize(self) -> None:
        self._check(self.lib.nova_finalize(self.h), "nova_finalize")

    def query_sms(self):
        t, g, n = A.I32(), A.I32(), A.I32()
        self._check(self.lib.nova_query_sms(self.h, C.byref(t), C.byref(g), C.byref(n)), "nova_query_sms")
        return t.value, g.value, n.value

    def set_partition(self, mode=ADAPTIVE, sm_decode_dv=72, sm_decode_dp=72, sm_op_dv=48, sm_op_dp=48, sm_min=16,
                      alpha_dv=8.0, alpha_dp=8.0, b_max=0, pf_threshold=5, sm_dv_floor=0,
                      chunk_budget=128, front_regroup=0) -> A.PartitionPolicy:
        p = A.PartitionPolicy(mode, sm_decode_dv, sm_decode_dp, sm_op_dv, sm_op_dp, sm_min, alpha_dv, alpha_dp, b_max,
                              pf_threshold, sm_dv_floor, chunk_budget, front_regroup)
        out = A.PartitionPolicy()
        self._check(self.lib.nova_set_partition(self.h, C.byref(p), C.byref(out)), "nova_set_partition")
        return out

    def set_frontier(self, points, window: int = 16) -> None:
        """points: (s_v, s_p, e2e_ms, thr_rps, on_frontier) tuples (nova_plan's 'points')."""
        arr = (A.PlanPoint * len(points))(*[A.PlanPoint(int(a), int(b), float(c), float(d), int(f), 0)
                                            for a, b, c, d, f in points])
        self._check(self.lib.nova_set_frontier(self.h, arr, len(points), window), "nova_set_frontier")

    # -------------------------------------------------------------- serving
    def submit(self, pixels: np.ndarray | None, prompt_ids, gen_len: int, arrival_ns: int = 0, grid=None,
               vis_scale: float = 1.0, pre_scale: float = 1.0) -> int:
        r = A.Request()
        if pixels is not None:
            pix = np.ascontiguousarray(pixels, dtype=np.uint16)
            self._keep_alive = pix
            r.pixels_bf16 = pix.ctypes.data
            r.height, r.width = int(pix.shape[1]), int(pix.shape[2])
        else:  # Sim backend: only the image size matters
            gh, gw = grid
            r.height, r.width = gh * self.shape.patch, gw * self.shape.patch
        ids = np.ascontiguousarray(prompt_ids, dtype=np.int32)
        r.prompt_ids = ids.ctypes.data if len(ids) else None
        r.n_prompt = len(ids)
        r.gen_len = int(gen_len)
        r.arrival_ns = int(arrival_ns)
        r.sim_vision_scale, r.sim_prefill_scale = vis_scale, pre_scale
        rid = A.U64()
        rc = self.lib.nova_submit(self.h, C.byref(r), C.byref(rid))
        if rc == -4:
            return -1      # NOVA_E_AGAIN
        self._check(rc, "nova_submit")
        return rid.value

    def step(self, max_wait_us: int = 0) -> A.StepInfo:
        info = A.StepInfo()
        self._check(self.lib.nova_step(self.h, int(max_wait_us), C.byref(info)), "nova_step")
        return info

    def poll_tokens(self, cap: int = 4096) -> list:
        buf = (A.Token * cap)()
        n = A.I32()
        self._check(self.lib.nova_poll_tokens(self.h, buf, cap, C.byref(n)), "nova_poll_tokens")
        return [(buf[i].req_id, buf[i].index, buf[i].token, buf[i].t_emit_ns, buf[i].flags) for i in range(n.value)]

    def stats(self, rid: int) -> dict:
        s = A.ReqStats()
        self._check(self.lib.nova_request_stats(self.h, rid, C.byref(s)), "nova_request_stats")
        return {f: getattr(s, f) for f, _ in A.ReqStats._fields_}

    def release(self, rid: int) -> None:
        self._check(self.lib.nova_release_request(self.h, rid), "nova_release_request")

    def decision_log(self) -> list:
        """Retained records (the log is a bounded ring: records before nova_decision_log_base are gone)."""
        out, start = [], self.lib.nova_decision_log_base(self.h)
        buf = (A.LogRecord * 4096)()
        while True:
            n, tot = A.I32(), A.I64()
            self._check(self.lib.nova_decision_log(self.h, start, buf, 4096, C.byref(n), C.byref(tot)), "log")
            for i in range(n.value):
                r = buf[i]
                out.append((r.tick, r.is_event, r.kind, r.ctx, r.s_dec, tuple(r.ids[:r.n_ids]), r.t_ns))
            start += n.value
            if start >= tot.value or n.value == 0:
                return out

    def debug_logits(self, rid: int, index: int) -> np.ndarray:
        v = self.shape.vocab
        out = np.empty(v, np.float32)
        self._check(self.lib.nova_debug_logits(self.h, rid, index, out.ctypes.data_as(C.POINTER(A.F32)), v),
                    "nova_debug_logits")
        return out

    def force_tokens(self, rid: int, tokens) -> None:
        a = np.ascontiguousarray(tokens, dtype=np.int32)
        self._check(self.lib.nova_debug_force_tokens(self.h, rid, a.ctypes.data_as(C.POINTER(A.I32)), len(a)),
                    "nova_debug_force_tokens")

    def time_pass(self, stage: int, s: int, gh=52, gw=94, n_prompt=64, B=1, ctx=1334, corun=0, iters=3):
        out = (A.F64 * 2)()
        self._check(self.lib.nova_time_pass(self.h, stage, s, gh, gw, n_prompt, B, ctx, corun, iters, out),
                    "nova_time_pass")
        return out[0], out[1]

    def debug_read_buffer(self, name: str, nbytes: int) -> bytes:
        """Raw bytes of an internal decode workspace buffer (nova_debug_read_buffer)."""
        buf = C.create_string_buffer(nbytes)
        self._check(self.lib.nova_debug_read_buffer(self.h, name.encode(), buf, nbytes), "nova_debug_read_buffer")
        return buf.raw

    def kernel_timing(self, every_n: int) -> None:
        self._check(self.lib.nova_kernel_timing(self.h, every_n), "nova_kernel_timing")

    def kernel_stats(self) -> dict:
        """{class: (device ms, algorithmic work, launches)} for the NOVA_K_* classes."""
        out = {}
        buf = (A.F64 * 3)()
        for cls, name in enumerate(KERNEL_CLASSES):
            self._check(self.lib.nova_kernel_stats(self.h, cls, buf), "nova_kernel_stats")
            out[name] = (buf[0], buf[1], int(buf[2]))
        return out

    def kernel_stats_sm(self) -> dict:
        """{class: SM-share-weighted device ms} (partition-normalized time, include/nova.h)."""
        out = {}
        v = A.F64(0.0)
        for cls, name in enumerate(KERNEL_CLASSES):
            self._check(self.lib.nova_kernel_stats_sm(self.h, cls, C.byref(v)), "nova_kernel_stats_sm")
            out[name] = v.value
        return out

    def kernel_stats_reset(self) -> None:
        self._check(self.lib.nova_kernel_stats_reset(self.h), "nova_kernel_stats_reset")

    def sim_set_curves(self, splits, t_v, t_p, t_d_dv, t_d_dp, t_v_solo, t_p_solo, t_d_solo, beta=0.0,
                       total_sms=148, granularity=8):
        n = len(splits)
        s = (A.I32 * n)(*[int(x) for x in splits])
        ts = [(A.I64 * n)(*[int(x) for x in xs]) for xs in (t_v, t_p, t_d_dv, t_d_dp)]
        self._sc_keep = [s] + ts
        ptr = lambda a: C.cast(a, C.POINTER(A.I64))
        sc = A.SimCurves(n, C.cast(s, C.POINTER(A.I32)), ptr(ts[0]), ptr(ts[1]), ptr(ts[2]), ptr(ts[3]),
                         int(t_v_solo), int(t_p_solo), int(t_d_solo), float(beta), total_sms, granularity)
        self._check(self.lib.nova_sim_set_curves(self.h, C.byref(sc)), "nova_sim_set_curves")


# ------------------------------------------------------------------ pure host functions
def nova_adaptive_sm(sm_op, sm_min, alpha, n_pending, granularity) -> int:
    return lib().nova_adaptive_sm(sm_op, sm_min, float(alpha), n_pending, granularity)


def nova_next_logical_layer(cur, K, L) -> int:
    return lib().nova_next_logical_layer(cur, K, L)


def nova_offload_floor(s, t_v, t_h2d_ms) -> int:
    n = len(s)
    return lib().nova_offload_floor((A.I32 * n)(*s), (A.F64 * n)(*[float(x) for x in t_v]), n, float(t_h2d_ms))


def nova_required_bandwidth(nbytes, forward_s, L, K) -> float:
    return lib().nova_required_bandwidth(float(nbytes), float(forward_s), L, K)


def nova_plan(s, t_v, t_p, t_d_dv, t_d_dp, gen_len, tau=2.5, t_d_full=0.0) -> dict:
    n = len(s)
    S = (A.I32 * n)(*s)
    arr = lambda xs: (A.F64 * n)(*[float(x) for x in xs])
    tv, tp, tdv, tdp = arr(t_v), arr(t_p), arr(t_d_dv), arr(t_d_dp)
    fp = lambda a: C.cast(a, C.POINTER(A.F64))
    cv = A.Curves(n, C.cast(S, C.POINTER(A.I32)), fp(tv), fp(tp), fp(tdv), fp(tdp), float(t_d_full))
    pts = (A.PlanPoint * (n * n))()
    nout, smin = A.I32(), A.I32()
    best = A.PlanPoint()
    adv, adp = A.F64(), A.F64()
    rc = lib().nova_plan(C.byref(cv), float(gen_len), float(tau), pts, n * n, C.byref(nout), C.byref(best),
                         C.byref(smin), C.byref(adv), C.byref(adp))
    if rc != 0:
        raise NovaError(f"nova_plan -> {rc}")
    P = [(p.s_v, p.s_p, p.e2e_ms, p.thr_rps, p.on_frontier) for p in pts[:nout.value]]
    return {"points": P, "best": (best.s_v, best.s_p, best.e2e_ms, best.thr_rps), "sm_min": smin.value,
            "alpha_dv": adv.value, "alpha_dp": adp.value}
