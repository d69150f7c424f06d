"""Python binding of include/nova_ops.h: same names, argument marshalling only.

Tensors are torch CUDA tensors (device memory plumbing); every computation runs
in libnova.so kernels on the current torch stream.
"""
from __future__ import annotations

import torch

from ._lib import lib, check

(EPI_BF16, EPI_BF16_QGELU, EPI_BF16_GELU, EPI_BF16_SILUMUL, EPI_F32_RESID, EPI_F32_STORE, EPI_QKV_ROPE_KV,
 EPI_F32_ARGMAX) = range(8)
XM_BF16, XM_F32, XM_NORM_BF16, XM_NORM_F32 = range(4)


def _p(t):
    return None if t is None else t.data_ptr()


def _s(stream=None):
    return (stream or torch.cuda.current_stream()).cuda_stream


def nova_op_gemm(A, W, C, bias, M, N, K, epi, max_ctas=148, lda=None, ldw=None, ldc=None, stream=None):
    check(lib().nova_op_gemm(_p(A), lda or A.stride(0), _p(W), ldw or W.stride(0), _p(C), ldc or C.stride(0),
                             _p(bias), M, N, K, epi, max_ctas, _s(stream)), "gemm")


def nova_op_gemm_fold(A, W, C, bias, M, N, K, epi, ngamma=None, nxout=None, nss=None, rscale=None, max_ctas=148,
                      stream=None):
    """nova_op_gemm with the RMSNorm fold (include/nova_ops.h): nxout / nss outputs of a NOVA_EPI_F32_RESID
    GEMM, or the rscale [M] row scales (nova_op_fold_rows) of a NOVA_EPI_BF16(_SILUMUL) GEMM."""
    check(lib().nova_op_gemm_fold(_p(A), A.stride(0), _p(W), W.stride(0), _p(C), C.stride(0), _p(bias), M, N, K, epi,
                                  max_ctas, _p(ngamma), _p(nxout), nxout.stride(0) if nxout is not None else 0,
                                  _p(nss), nss.stride(0) if nss is not None else 0, _p(rscale), _s(stream)), "gemm_fold")


def nova_op_gemm_rope2d(A, W, C, bias, M, N, K, qk_cols, gw, merge, theta, max_ctas=148, stream=None):
    import ctypes as Ct
    check(lib().nova_op_gemm_rope2d(_p(A), A.stride(0), _p(W), W.stride(0), _p(C), C.stride(0), _p(bias), M, N, K,
                                    qk_cols, gw, merge, Ct.c_float(theta), max_ctas, _s(stream)), "gemm_rope2d")


def nova_op_fold_rows(ss, d, eps, rscale, M, stream=None):
    import ctypes as Ct
    check(lib().nova_op_fold_rows(_p(ss), ss.stride(0), d, Ct.c_float(eps), _p(rscale), M, _s(stream)), "fold_rows")


def nova_op_rms_prep(x, gamma, y, ss, M, d, stream=None):
    check(lib().nova_op_rms_prep(_p(x), x.stride(0), _p(gamma), _p(y), y.stride(0), _p(ss), ss.stride(0), M, d,
                                 _s(stream)), "rms_prep")


def nova_op_gemm_mode(mode: int) -> int:
    """0 = automatic tile choice, 1 = single-CTA tiles only, 2 = CTA-pair tiles only; returns the previous mode."""
    return lib().nova_op_gemm_mode(mode)


def nova_op_gemm_config(M: int, N: int, K: int) -> int:
    """Tile the current mode picks for this shape: pair * 1000 + BN."""
    return lib().nova_op_gemm_config(M, N, K)


def nova_op_gemv(X, W, Y, bias, N, K, B, epi, x_f32=None, ldx=None, ldy=None, stream=None):
    xf = int(X.dtype == torch.float32) if x_f32 is None else x_f32
    check(lib().nova_op_gemv(_p(X), xf, ldx or X.stride(0), _p(W), N, K, _p(Y), ldy or Y.stride(0), _p(bias), B,
                             epi, _s(stream)), "gemv")


_ws_cache = {}


def nova_op_gemv_tma(X, W, Y, bias, N, K, B, epi, ldx=None, ldy=None, max_ctas=0, stream=None):
    dev = X.device
    if dev not in _ws_cache:
        _ws_cache[dev] = (torch.empty(16 * 16 * 160000, dtype=torch.float32, device=dev),
                          torch.zeros(8192, dtype=torch.int32, device=dev))
    ws, tk = _ws_cache[dev]
    check(lib().nova_op_gemv_tma(_p(X), ldx or X.stride(0), _p(W), N, K, _p(Y), ldy or Y.stride(0), _p(bias), B,
                                 epi, _p(ws), _p(tk), max_ctas, _s(stream)), "gemv_tma")


def nova_op_flash_attn(qkv, out, S, H, KV, hd, causal, max_ctas=0, stream=None):
    check(lib().nova_op_flash_attn(_p(qkv), qkv.stride(0), _p(out), out.stride(0), S, H, KV, hd, int(causal),
                                   max_ctas, _s(stream)), "flash_attn")


def nova_op_flash_attn_mma(qkv, out, S, H, KV, hd, causal, stream=None):
    check(lib().nova_op_flash_attn_mma(_p(qkv), qkv.stride(0), _p(out), out.stride(0), S, H, KV, hd, int(causal),
                                       _s(stream)), "flash_attn_mma")


def nova_op_decode_attn(qkv, out, kv_pool, layer, n_pages, H, KV, hd, block_tables, rows, B, max_ctx, ws,
                        tickets=None, max_ctas=0, stream=None):
    if tickets is None:
        tickets = torch.zeros(B * KV, dtype=torch.int32, device=qkv.device)
    check(lib().nova_op_decode_attn(_p(qkv), qkv.stride(0), _p(out), out.stride(0), _p(kv_pool), layer, n_pages,
                                    H, KV, hd, _p(block_tables), block_tables.shape[1], _p(rows), B, max_ctx, _p(ws),
                                    _p(tickets), max_ctas, _s(stream)), "decode_attn")


def nova_op_gemv_fused(X, x_mode, W, Y, bias, N, K, B, epi, gamma=None, eps=0.0, H=0, KV=0, hd=0, theta=0.0,
                       rows=None, kv_pool=None, layer=0, n_pages=0, block_tables=None, keys=None, ldx=None, ldy=None,
                       stream=None):
    import ctypes as C
    check(lib().nova_op_gemv_fused(_p(X), x_mode, ldx or X.stride(0), _p(W), N, K, _p(Y), ldy or Y.stride(0),
                                   _p(bias), B, epi, _p(gamma), C.c_float(eps), H, KV, hd, C.c_float(theta), _p(rows),
                                   _p(kv_pool), layer, n_pages, _p(block_tables),
                                   0 if block_tables is None else block_tables.shape[1], _p(keys), _s(stream)),
          "gemv_fused")


def nova_op_argmax_finalize(keys, n, out_tok, rows=None, last_tok=None, single_slot=-1, stream=None):
    check(lib().nova_op_argmax_finalize(_p(keys), n, _p(out_tok), _p(rows), _p(last_tok), single_slot, _s(stream)),
          "argmax_finalize")


def nova_op_layernorm(x, gamma, beta, y, M, d, eps, stream=None):
    check(lib().nova_op_layernorm(_p(x), x.stride(0), _p(gamma), _p(beta), _p(y), y.stride(0), M, d, eps,
                                  _s(stream)), "layernorm")


def nova_op_rmsnorm(x, gamma, y, M, d, eps, y_mode=None, stream=None):
    """y_mode: 0 bf16, 1 f32 (default from y's dtype), 2 bf16 hi rows then bf16 lo rows (y [2M][d])."""
    mode = int(y.dtype == torch.float32) if y_mode is None else y_mode
    check(lib().nova_op_rmsnorm(_p(x), x.stride(0), _p(gamma), _p(y), mode, y.stride(0), M, d, eps, _s(stream)),
          "rmsnorm")


def nova_op_patchify(pix, P, T, merge, X0, stream=None):
    Cc, H, W = pix.shape
    check(lib().nova_op_patchify(_p(pix), Cc, H, W, P, T, merge, _p(X0), _s(stream)), "patchify")


def nova_op_vit_rope(qkv, N, heads, hd, gw, merge, theta, stream=None):
    check(lib().nova_op_vit_rope(_p(qkv), N, heads, hd, gw, merge, theta, _s(stream)), "vit_rope")


def nova_op_llm_rope_kv(qkv, nrows, H, KV, hd, theta, sec0, sec1, pos3, rows, slot, ctx0, kv_pool, layer, n_pages,
                        block_tables, stream=None):
    check(lib().nova_op_llm_rope_kv(_p(qkv), qkv.stride(0), nrows, H, KV, hd, theta, sec0, sec1, _p(pos3),
                                    0 if pos3 is None else pos3.stride(0), _p(rows), slot, ctx0, _p(kv_pool), layer,
                                    n_pages, _p(block_tables), block_tables.shape[1], _s(stream)), "llm_rope_kv")


def nova_op_embed(table, d, ids, rows, last_tok, out, n, stream=None):
    check(lib().nova_op_embed(_p(table), d, _p(ids), _p(rows), _p(last_tok), _p(out), out.stride(0), n,
                              _s(stream)), "embed")


def nova_op_argmax(logits, V, n, out_tok, rows=None, last_tok=None, single_slot=-1, stream=None):
    check(lib().nova_op_argmax(_p(logits), logits.stride(0), V, n, _p(out_tok), _p(rows), _p(last_tok),
                               single_slot, _s(stream)), "argmax")


def nova_op_block_weights(W, Wb, N, K, stream=None):
    check(lib().nova_op_block_weights(_p(W), _p(Wb), N, K, _s(stream)), "block_weights")


def nova_op_gemv_stream(X, Wb, Y, bias, N, K, B, epi, X_lo=None, keys=None, max_ctas=0, ldx=None, ldy=None,
                        stream=None):
    dev = X.device
    if dev not in _ws_cache:
        _ws_cache[dev] = (torch.empty(16 * 16 * 160000, dtype=torch.float32, device=dev),
                          torch.zeros(8192, dtype=torch.int32, device=dev))
    ws, tk = _ws_cache[dev]
    check(lib().nova_op_gemv_stream(_p(X), _p(X_lo), ldx or X.stride(0), _p(Wb), N, K, _p(Y), ldy or Y.stride(0),
                                    _p(bias), B, epi, _p(ws), _p(tk), _p(keys), max_ctas, _s(stream)), "gemv_stream")


def nova_op_gemv_umma(X, Wb, Y, bias, N, K, B, epi, X_lo=None, keys=None, max_ctas=0, ldx=None, ldy=None,
                      norm_hid=None, norm_eps=0.0, ngamma=None, nxout=None, stream=None):
    dev = X.device
    if dev not in _ws_cache:
        _ws_cache[dev] = (torch.empty(16 * 16 * 160000, dtype=torch.float32, device=dev),
                          torch.zeros(8192, dtype=torch.int32, device=dev))
    ws, tk = _ws_cache[dev]
    check(lib().nova_op_gemv_umma(_p(X), _p(X_lo), ldx or X.stride(0), _p(Wb), N, K, _p(Y), ldy or Y.stride(0),
                                  _p(bias), B, epi, _p(ws), _p(tk), _p(keys), max_ctas, _p(norm_hid), float(norm_eps),
                                  _p(ngamma), _p(nxout), nxout.stride(0) if nxout is not None else 0,
                                  _s(stream)), "gemv_umma")


def nova_op_gemv_umma_qkv(X, Wb, Q, bias, N, K, B, norm_hid, norm_eps, H, KV, hd, theta, rows, kv_pool, layer,
                          n_pages, block_tables, max_ctas=0, stream=None):
    import ctypes as C
    dev = X.device
    if dev not in _ws_cache:
        _ws_cache[dev] = (torch.empty(16 * 16 * 160000, dtype=torch.float32, device=dev),
                          torch.zeros(8192, dtype=torch.int32, device=dev))
    ws, tk = _ws_cache[dev]
    check(lib().nova_op_gemv_umma_qkv(_p(X), X.stride(0), _p(Wb), N, K, _p(Q), Q.stride(0), _p(bias), B,
                                      _p(norm_hid), C.c_float(norm_eps), H, KV, hd, C.c_float(theta), _p(rows),
                                      _p(kv_pool), layer, n_pages, _p(block_tables), block_tables.shape[1], _p(ws),
                                      _p(tk), max_ctas, _s(stream)), "gemv_umma_qkv")


def nova_op_scale_rows_bf16(x, gamma, y, M, d, stream=None):
    check(lib().nova_op_scale_rows_bf16(_p(x), x.stride(0), _p(gamma), _p(y), y.stride(0), M, d, _s(stream)),
          "scale_rows_bf16")


def nova_op_gemv_umma_splits(N: int, K: int, epi: int) -> int:
    return lib().nova_op_gemv_umma_splits(N, K, epi)


def nova_op_chunk_attn(qkv, out, C, c0, H, KV, hd, kv_pool, layer, n_pages, block_table_row, stream=None):
    check(lib().nova_op_chunk_attn(_p(qkv), qkv.stride(0), _p(out), out.stride(0), C, c0, H, KV, hd, _p(kv_pool), layer,
                                   n_pages, _p(block_table_row), _s(stream)), "chunk_attn")


def nova_op_decode_attn_p(qkv, out, kv_pool, layer, n_pages, H, KV, hd, block_tables, rows, B, max_ctx, ws, tickets,
                          mch, max_ctas=0, stream=None):
    check(lib().nova_op_decode_attn_p(_p(qkv), qkv.stride(0), _p(out), out.stride(0), _p(kv_pool), layer, n_pages, H,
                                      KV, hd, _p(block_tables), block_tables.shape[1], _p(rows), B, max_ctx, _p(ws),
                                      _p(tickets), mch, max_ctas, _s(stream)), "decode_attn_p")
