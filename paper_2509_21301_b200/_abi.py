"""ctypes mirror of include/nova.h (structs and function signatures)."""
from __future__ import annotations

import ctypes as C

I32, I64, U64, F32, F64, P = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p


class ModelConfig(C.Structure):
    _fields_ = [(n, I32) for n in ("vit_depth", "vit_dim", "vit_heads", "vit_mlp", "patch", "temporal_patch",
                                   "merge", "in_ch", "llm_layers", "llm_dim", "llm_heads", "llm_kv_heads",
                                   "head_dim", "llm_ffn", "vocab", "tie_embed")] + \
              [("mrope_section", I32 * 3), ("vit_theta", F32), ("llm_theta", F32), ("ln_eps", F32), ("rms_eps", F32)]


class EngineConfig(C.Structure):
    _fields_ = [(n, I32) for n in ("backend", "device", "max_requests", "max_decode_batch", "kv_pages",
                                   "max_patches", "max_prompt", "max_gen", "vit_resident_layers",
                                   "use_green_ctx", "debug_keep_logits", "finished_retention")]


class Buffers(C.Structure):
    _fields_ = [("weights_dev", P), ("weights_bytes", U64), ("kv_dev", P), ("kv_bytes", U64),
                ("workspace_dev", P), ("workspace_bytes", U64)]


class Request(C.Structure):
    _fields_ = [("pixels_bf16", P), ("height", I32), ("width", I32), ("prompt_ids", P), ("n_prompt", I32),
                ("gen_len", I32), ("arrival_ns", I64), ("user_tag", U64), ("sim_vision_scale", F32),
                ("sim_prefill_scale", F32)]


class PartitionPolicy(C.Structure):
    _fields_ = [("mode", I32), ("sm_decode_dv", I32), ("sm_decode_dp", I32), ("sm_op_dv", I32),
                ("sm_op_dp", I32), ("sm_min", I32), ("alpha_dv", F32), ("alpha_dp", F32), ("b_max", I32),
                ("pf_threshold", I32), ("sm_dv_floor", I32), ("chunk_budget", I32),
                ("front_regroup", I32)]


class StepInfo(C.Structure):
    _fields_ = [(n, I32) for n in ("events", "dispatched", "n_pending", "sm_decode", "context", "decode_batch",
                                   "active", "finished")] + [("now_ns", I64)]


class Token(C.Structure):
    _fields_ = [("req_id", U64), ("index", I32), ("token", I32), ("t_emit_ns", I64), ("flags", I32), ("pad", I32)]


class ReqStats(C.Structure):
    _fields_ = [(n, I64) for n in ("arrival", "vis_start", "vis_end", "pre_start", "pre_end", "first_tok",
                                   "last_tok")] + [(n, I32) for n in ("split_at_vis", "split_at_pre", "n_tokens",
                                                                      "finished")]


class LogRecord(C.Structure):
    _fields_ = [("t_ns", I64), ("tick", I32), ("is_event", I32), ("kind", I32), ("ctx", I32), ("s_dec", I32),
                ("n_ids", I32), ("ids", U64 * 16)]


class Curves(C.Structure):
    _fields_ = [("n", I32), ("s", C.POINTER(I32)), ("t_v", C.POINTER(F64)), ("t_p", C.POINTER(F64)),
                ("t_d_dv", C.POINTER(F64)), ("t_d_dp", C.POINTER(F64)), ("t_d_full", F64)]


class PlanPoint(C.Structure):
    _fields_ = [("s_v", I32), ("s_p", I32), ("e2e_ms", F64), ("thr_rps", F64), ("on_frontier", I32), ("pad", I32)]


class SimCurves(C.Structure):
    _fields_ = [("n", I32), ("s", C.POINTER(I32)), ("t_v", C.POINTER(I64)), ("t_p", C.POINTER(I64)),
                ("t_d_dv", C.POINTER(I64)), ("t_d_dp", C.POINTER(I64)), ("t_v_solo", I64), ("t_p_solo", I64),
                ("t_d_solo", I64), ("beta", F64), ("total_sms", I32), ("granularity", I32)]


R = I32  # nova_status
E = P    # nova_engine*
ENGINE_SIGNATURES = {
    "nova_query_memory": (R, [C.POINTER(ModelConfig), C.POINTER(EngineConfig), C.POINTER(U64), C.POINTER(U64),
                              C.POINTER(U64), C.POINTER(U64)]),
    "nova_create": (R, [C.POINTER(ModelConfig), C.POINTER(EngineConfig), C.POINTER(Buffers), C.POINTER(E)]),
    "nova_load_tensor": (R, [E, C.c_char_p, P, U64, I32]),
    "nova_finalize": (R, [E]),
    "nova_destroy": (R, [E]),
    "nova_last_error": (C.c_char_p, [E]),
    "nova_query_sms": (R, [E, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
    "nova_submit": (R, [E, C.POINTER(Request), C.POINTER(U64)]),
    "nova_set_partition": (R, [E, C.POINTER(PartitionPolicy), C.POINTER(PartitionPolicy)]),
    "nova_set_frontier": (R, [E, C.POINTER(PlanPoint), I32, I32]),
    "nova_step": (R, [E, I64, C.POINTER(StepInfo)]),
    "nova_poll_tokens": (R, [E, C.POINTER(Token), I32, C.POINTER(I32)]),
    "nova_request_stats": (R, [E, U64, C.POINTER(ReqStats)]),
    "nova_decision_log": (R, [E, I64, C.POINTER(LogRecord), I32, C.POINTER(I32), C.POINTER(I64)]),
    "nova_decision_log_base": (I64, [E]),
    "nova_release_request": (R, [E, U64]),
    "nova_debug_logits": (R, [E, U64, I32, C.POINTER(F32), I32]),
    "nova_debug_read_buffer": (R, [E, C.c_char_p, C.c_void_p, U64]),
    "nova_front_switches": (I64, [E]),
    "nova_debug_force_tokens": (R, [E, U64, C.POINTER(I32), I32]),
    "nova_time_pass": (R, [E, I32, I32, I32, I32, I32, I32, I32, I32, I32, C.POINTER(F64)]),
    "nova_plan": (R, [C.POINTER(Curves), F64, F64, C.POINTER(PlanPoint), I32, C.POINTER(I32), C.POINTER(PlanPoint),
                      C.POINTER(I32), C.POINTER(F64), C.POINTER(F64)]),
    "nova_adaptive_sm": (I32, [I32, I32, F64, I32, I32]),
    "nova_next_logical_layer": (I32, [I32, I32, I32]),
    "nova_required_bandwidth": (F64, [F64, F64, I32, I32]),
    "nova_offload_floor": (I32, [C.POINTER(I32), C.POINTER(F64), I32, F64]),
    "nova_sim_set_curves": (R, [E, C.POINTER(SimCurves)]),
    "nova_kernel_timing": (R, [E, I32]),
    "nova_kernel_stats": (R, [E, I32, C.POINTER(F64)]),
    "nova_kernel_stats_sm": (R, [E, I32, C.POINTER(F64)]),
    "nova_kernel_stats_reset": (R, [E]),
    "nova_launch_count": (U64, []),
}


def declare(lb) -> None:
    for name, (res, args) in ENGINE_SIGNATURES.items():
        fn = getattr(lb, name)   # AttributeError = the library lacks a declared symbol
        fn.argtypes = args
        fn.restype = res
