"""Test infrastructure (not collected).  Debug: tiny end-to-end decode with the fused kernel stopped at phase k (per-op path finishes),
compared with the oracle.  python scripts/dbg_fused.py k1 k2 ...  (runs each k in a subprocess)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import numpy as np
    from synth import TINY, gen_weights, tiny_request
    from oracle import vlm as V
    from paper_2509_21301_b200 import engine as E
    seed = json.load(open(os.path.join(ROOT, "tests", "golden", "tiny_seed.json")))["seed"]
    bits = gen_weights(TINY, seed)
    req = tiny_request(TINY, seed)
    eng = E.Engine(TINY, E.EngineOptions(max_requests=4, kv_pages=16, max_patches=64, max_prompt=16, max_gen=16,
                                         debug_keep_logits=1))
    eng.load_weights(bits)
    eng.finalize()
    eng.set_partition(E.SERIAL)
    rid = eng.submit(req.pixels, req.prompt_ids, req.gen_len)
    while eng.step(2000).finished < 1:
        pass
    toks = [t for _, t in sorted((i, t) for r, i, t, _, _ in eng.poll_tokens() if r == rid)]
    logits = np.stack([eng.debug_logits(rid, k) for k in range(req.gen_len)])
    ref = V.generate(V.OracleWeights(bits, np.float32), req.pixels, req.prompt_ids, req.gen_len, TINY)
    err = np.abs(logits - ref["logits"]).max(axis=1)
    print(json.dumps({"stop": os.environ.get("NOVA_DEC_FUSED_STOP"), "fused": os.environ.get("NOVA_DEC_FUSED"),
                      "ok": toks == ref["tokens"].tolist(), "err_per_step": [round(float(x), 4) for x in err]}),
          flush=True)
    eng.close()


def halt_check(stop: int):
    """NOVA_DEC_FUSED_STOP=stop + HALT: the engine fails right after the first (partial) fused decode
    kernel; compare its buffers with numpy on the same bits (layer 0)."""
    import numpy as np
    from synth import TINY, gen_weights, tiny_request
    from synth.weights import bf16_bits_to_f32 as b2f, f32_to_bf16_bits as f2b
    from paper_2509_21301_b200 import engine as E
    s = TINY
    seed = json.load(open(os.path.join(ROOT, "tests", "golden", "tiny_seed.json")))["seed"]
    bits = gen_weights(s, seed)
    req = tiny_request(s, seed)
    eng = E.Engine(s, E.EngineOptions(max_requests=4, kv_pages=16, max_patches=64, max_prompt=16, max_gen=16,
                                       debug_keep_logits=1))
    eng.load_weights(bits)
    eng.finalize()
    eng.set_partition(E.SERIAL)
    rid = eng.submit(req.pixels, req.prompt_ids, req.gen_len)
    tok0 = None
    try:
        for _ in range(200):
            eng.step(2000)
            for r, i, t, _, _ in eng.poll_tokens():
                if i == 0:
                    tok0 = t
    except Exception as ex:  # the halt
        print("halted:", str(ex)[:80])
    Bm = eng.opts.max_decode_batch if hasattr(eng, "opts") else 16
    D, H, KV, hd = s.llm_dim, s.llm_heads, s.llm_kv_heads, s.head_dim
    ldq = (H + 2 * KV) * hd

    def rd(name, shape, dt):
        n = int(np.prod(shape)) * np.dtype(dt).itemsize
        a = np.frombuffer(eng.debug_read_buffer(name, n), dtype=dt).reshape(shape)
        return b2f(a) if dt == np.uint16 else a
    W = {k: b2f(v) for k, v in bits.items()}
    pre = "model.language_model.layers.0."
    h0 = W["model.language_model.embed_tokens.weight"][tok0].astype(np.float64)
    g1 = W[pre + "input_layernorm.weight"]
    xg = b2f(f2b((h0 * g1).astype(np.float32))).astype(np.float64)
    inv = 1.0 / np.sqrt((h0 * h0).mean() + s.rms_eps)
    wq = np.concatenate([W[pre + "self_attn.%s_proj.weight" % n] for n in "qkv"], 0)
    bq = np.concatenate([W[pre + "self_attn.%s_proj.bias" % n] for n in "qkv"], 0)
    qkv_ref = inv * (wq @ xg) + bq
    out = {"stop": stop, "tok0": tok0}
    if stop >= 2:
        qkvf = rd("dec_qkvf", (1, ldq), np.float32)[0]
        out["qkv_maxerr"] = float(np.abs(qkvf - qkv_ref).max())
        out["qkv_scale"] = float(np.abs(qkv_ref).max())
    if stop >= 4:
        attn = rd("dec_attn", (1, H * hd), np.uint16)[0].astype(np.float64)
        hid = rd("dec_hid", (1, D), np.float32)[0]
        hid_ref = h0 + W[pre + "self_attn.o_proj.weight"] @ attn
        out["hid_maxerr"] = float(np.abs(hid - hid_ref).max())
        out["hid_scale"] = float(np.abs(hid_ref).max())
        out["hid_head"] = [round(float(x), 4) for x in hid[:6]]
        out["ref_head"] = [round(float(x), 4) for x in hid_ref[:6]]
        d = np.abs(hid - hid_ref)
        out["bad_cols"] = [int(i) for i in np.nonzero(d > 1e-2)[0][:20]]
        out["h0_head"] = [round(float(x), 4) for x in h0[:6]]
        out["attn_absmax"] = float(np.abs(attn).max())
        out["hid_minus_h0_max"] = float(np.abs(hid - h0).max())
        xg2 = rd("dec_xg", (1, D), np.uint16)[0]
        g2 = W[pre + "post_attention_layernorm.weight"]
        out["xg_vs_hid_g2"] = float(np.abs(xg2 - hid * g2).max())
        ss = rd("dec_ss", (1, 4), np.float32)[0]
        out["ss"] = [float(x) for x in ss[:2]]
        out["ss_ref_from_hid"] = [float((hid[:64] ** 2).sum()), float((hid[64:128] ** 2).sum())]
    wo = rd("w_o0", (D, H * hd), np.uint16)
    wob = np.frombuffer(eng.debug_read_buffer("w_ob0", D * H * hd * 2), dtype=np.uint16)
    out["w_o0_matches_bits"] = bool(np.array_equal(wo, W[pre + "self_attn.o_proj.weight"]))
    out["w_ob0_nonzero"] = int(np.count_nonzero(wob))
    out["w_ob0_is_permutation"] = bool(np.array_equal(np.sort(wob), np.sort(bits[pre + "self_attn.o_proj.weight"].ravel())))
    if os.environ.get("NOVA_DEC_FUSED_DBG") == "1":
        q = rd("dec_qkvf", (16, ldq), np.float32)[15]
        for ph in range(5):
            print("dbg", [float(x) for x in q[ph * 12:ph * 12 + 12]])
        print("bar", rd("dec_qkvf", (16, ldq), np.float32)[14][:36].tolist())
        print("xtile", rd("dec_qkvf", (16, ldq), np.float32)[13][:18].tolist())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    elif len(sys.argv) > 1 and sys.argv[1] == "halt":
        halt_check(int(os.environ["NOVA_DEC_FUSED_STOP"]))
    else:
        for k in sys.argv[1:]:
            env = dict(os.environ)
            if k == "off":
                env["NOVA_DEC_FUSED"] = "0"
            else:
                env["NOVA_DEC_FUSED_STOP"] = k
            subprocess.run([sys.executable, __file__, "one"], env=env, timeout=120)

