"""End-to-end parity of the engine through the C ABI (GPU): the CUDA path vs the
oracle on the same generated weights and inputs (SURVEY.md §8(c) c1', c6).

- cfg 1 tiny VLM: greedy tokens identical, logits max-abs <= 3e-2 (BASELINE).
- co-execution == serial: tokens and f32 logits bitwise identical across SERIAL,
  STATIC splits, ADAPTIVE (also with front passes repartitioned every layer, §8(f) f4), the
  frontier-lookup controller and the paper's PF-Limit / Multi-Stream baselines on a
  20-request trace (BASELINE).
- offload: K = 2, 3, 4 physical ViT layers give bitwise the all-resident outputs over several
  vision passes, with a depth (7) that no K divides (the ring's slots rotate across passes).
- full width (reduced depth): 2B / 7B widths at the BASELINE image size (N = 4888),
  S = 1286, tokens teacher-forced, logits within tolerance.
"""
import json
import os
import time
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import vlm as V
from synth import TINY, Q2B, Q7B, gen_weights, tiny_request, make_request, reduced_depth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _engine(shape, bits, **kw):
    from paper_2509_21301_b200 import engine as E
    opts = dict(max_requests=24, max_decode_batch=16, kv_pages=256, max_patches=64, max_prompt=16, max_gen=16,
                debug_keep_logits=1)
    opts.update(kw)
    e = E.Engine(shape, E.EngineOptions(**opts))
    e.load_weights(bits)
    e.finalize()
    return e


def _run(e, reqs, forced=None, timeout_s=120):
    """Submit all requests at once, step until every one finished; tokens + logits per request."""
    ids = []
    for i, r in enumerate(reqs):
        rid = e.submit(r.pixels, r.prompt_ids, r.gen_len)
        assert rid > 0
        if forced is not None:
            e.force_tokens(rid, forced[i])
        ids.append(rid)
    t0 = time.time()
    while True:
        info = e.step(2000)
        if info.finished >= len(ids) + getattr(e, "_done_before", 0):
            break
        assert time.time() - t0 < timeout_s, "engine did not finish"
    e._done_before = info.finished
    toks = {}
    for rid, idx, tok, t, fl in e.poll_tokens(100000):
        toks.setdefault(rid, {})[idx] = tok
    out = []
    for rid, r in zip(ids, reqs):
        tk = [toks[rid][k] for k in range(r.gen_len)]
        lg = np.stack([e.debug_logits(rid, k) for k in range(r.gen_len)])
        out.append((tk, lg))
    return out


@pytest.fixture(scope="module")
def tiny_setup():
    seed = json.load(open(os.path.join(GOLD, "tiny_seed.json")))["seed"]
    bits = gen_weights(TINY, seed)
    req = tiny_request(TINY, seed)
    ref = V.generate(V.OracleWeights(bits, np.float32), req.pixels, req.prompt_ids, req.gen_len, TINY)
    return bits, req, ref


def test_tiny_end_to_end_parity(tiny_setup):
    from paper_2509_21301_b200 import engine as E
    bits, req, ref = tiny_setup
    e = _engine(TINY, bits)
    e.set_partition(E.SERIAL)
    (tk, lg), = _run(e, [req])
    assert tk == ref["tokens"].tolist()
    assert np.abs(lg - ref["logits"]).max() <= 3e-2
    e.close()


def test_coexec_bitwise_equals_serial(tiny_setup):
    from paper_2509_21301_b200 import engine as E
    bits, _, _ = tiny_setup
    reqs = [make_request(TINY, (4, 4) if i % 3 else (4, 6), 8 - (i % 4), 3 + (i % 6), 100 + i) for i in range(20)]
    results = {}
    e = _engine(TINY, bits)
    for name, pol in [("serial", dict(mode=E.SERIAL)),
                      ("static16", dict(mode=E.STATIC, sm_decode_dv=16, sm_decode_dp=16)),
                      # 8 decode SMs: large batches take the virtual-CTA decode attention (> 3 waves)
                      ("static8", dict(mode=E.STATIC, sm_decode_dv=8, sm_decode_dp=8)),
                      ("static56", dict(mode=E.STATIC, sm_decode_dv=56, sm_decode_dp=104)),
                      ("adaptive", dict(mode=E.ADAPTIVE, sm_op_dv=48, sm_op_dp=40, sm_min=8, alpha_dv=13.0,
                                        alpha_dp=10.0, b_max=5)),
                      ("adaptive_regroup", dict(mode=E.ADAPTIVE, sm_op_dv=48, sm_op_dp=40, sm_min=8, alpha_dv=13.0,
                                                alpha_dp=10.0, b_max=5, front_regroup=1)),   # f4: per layer
                      ("pf_limit", dict(mode=E.PF_LIMIT, pf_threshold=3)),
                      ("multi_stream", dict(mode=E.MULTI_STREAM)),
                      ("frontier", dict(mode=E.FRONTIER))]:
        if pol["mode"] == E.FRONTIER:   # two Pareto points: the lookup switches with the arrival rate
            e.set_frontier([(48, 40, 100.0, 5.0, 1), (16, 16, 140.0, 50.0, 1)], window=4)
        e.set_partition(**pol)
        results[name] = _run(e, reqs)
    base = results["serial"]
    for name, res in results.items():
        for (t0, l0), (t1, l1) in zip(base, res):
            assert t0 == t1, name
            assert np.array_equal(l0, l1), name
    # and each request matches the oracle
    for r, (tk, lg) in zip(reqs[:4], base[:4]):
        o = V.generate(V.OracleWeights(bits, np.float32), r.pixels, r.prompt_ids, r.gen_len, TINY, force_tokens=tk)
        assert np.abs(lg - o["logits"]).max() <= 3e-2
    e.close()


def test_offload_bitwise_equals_resident():
    from paper_2509_21301_b200 import engine as E
    s = replace(TINY, name="tiny-d7", vit_depth=7)   # 7 % K != 0 for every K below
    bits = gen_weights(s, 4)
    reqs = [make_request(s, (4, 4), 6, 4, 200 + i) for i in range(4)]   # 4 vision passes
    outs = []
    for K in (0, 2, 3, 4):
        e = _engine(s, bits, vit_resident_layers=K)
        e.set_partition(E.ADAPTIVE, sm_op_dv=32, sm_op_dp=32, sm_min=8, alpha_dv=8.0, alpha_dp=8.0)
        outs.append(_run(e, reqs))
        e.close()
    for o in outs[1:]:
        for (t0, l0), (t1, l1) in zip(outs[0], o):
            assert t0 == t1 and np.array_equal(l0, l1)


@pytest.mark.parametrize("base", [Q2B, Q7B], ids=["2b", "7b"])
def test_full_width_reduced_depth_parity(base):
    """BASELINE image size (grid 52x94, N = 4888) and S = 1286 at 2B / 7B width, depth 2+2."""
    from paper_2509_21301_b200 import engine as E
    s = reduced_depth(base, 2, 2)
    bits = gen_weights(s, 1)
    req = make_request(s, (52, 94), 64, 4, 1)
    e = _engine(s, bits, max_requests=2, kv_pages=64, max_patches=4888, max_prompt=64, max_gen=8)
    e.set_partition(E.ADAPTIVE, sm_op_dv=48, sm_op_dp=48, sm_min=16, alpha_dv=8.0, alpha_dp=8.0)
    (tk, lg), = _run(e, [req], timeout_s=300)
    ref = V.generate(V.OracleWeights(bits, np.float32), req.pixels, req.prompt_ids, req.gen_len, s,
                     force_tokens=tk)
    assert np.abs(lg - ref["logits"]).max() <= 5e-2 * max(1.0, np.abs(ref["logits"]).max() / 10)
    # where the oracle's choice is clear, the GPU's greedy token agrees
    for k in range(req.gen_len):
        srt = np.sort(ref["logits"][k])
        if srt[-1] - srt[-2] > 0.1:
            assert tk[k] == int(np.argmax(ref["logits"][k]))
    e.close()


@pytest.mark.parametrize("budget", [5, 128])
def test_chunked_prefill_mode_matches_oracle(tiny_setup, budget):
    """CHUNK (the paper's chunked-prefill baseline; R26): hybrid passes that batch
    prefill chunks with decode rows give the oracle's tokens and logits (<= 3e-2).  budget 5: the
    12-token tiny prefill takes 3-12 chunks, several of them sharing a batch with decode rows."""
    from paper_2509_21301_b200 import engine as E
    bits, req, ref = tiny_setup
    e = _engine(TINY, bits)
    e.set_partition(E.CHUNK, chunk_budget=budget, b_max=4)
    outs = _run(e, [req] * 4)
    for tk, lg in outs:
        assert tk == ref["tokens"].tolist()
        assert np.abs(lg - ref["logits"]).max() <= 3e-2
    log = e.decision_log()
    hyb = [r for r in log if not r[1] and r[2] == 4]   # NOVA_DEC_HYBRID
    assert hyb and sum(r[4] for r in hyb) == 4 * 12     # every prefill token in exactly one chunk
    if budget == 5:
        assert any(len(r[5]) > 1 for r in hyb)           # some chunk shared a batch with decode rows
    e.close()


def test_chunked_prefill_full_width_reduced_depth():
    """CHUNK at 2B width, BASELINE image size (S = 1286 -> 11 chunks of <= 128 tokens), depth 2+2:
    the chunked prefill's token-0 logits and the decode logits match the oracle (teacher-forced)."""
    from paper_2509_21301_b200 import engine as E
    s = reduced_depth(Q2B, 2, 2)
    bits = gen_weights(s, 1)
    req = make_request(s, (52, 94), 64, 4, 1)
    e = _engine(s, bits, max_requests=2, kv_pages=64, max_patches=4888, max_prompt=64, max_gen=8)
    e.set_partition(E.CHUNK, chunk_budget=128)
    (tk, lg), = _run(e, [req], timeout_s=300)
    ref = V.generate(V.OracleWeights(bits, np.float32), req.pixels, req.prompt_ids, req.gen_len, s,
                     force_tokens=tk)
    assert np.abs(lg - ref["logits"]).max() <= 5e-2 * max(1.0, np.abs(ref["logits"]).max() / 10)
    hyb = [r for r in e.decision_log() if not r[1] and r[2] == 4]
    assert len(hyb) == 11 and sum(r[4] for r in hyb) == 1286
    e.close()


def test_kernel_stats_partition_share(tiny_setup):
    """bench.py's partition-normalized roofline input (nova_kernel_stats_sm): every timed launch's ms is
    weighted by its pass's SM budget / total SMs -- under a static split with 16 decode SMs the decode
    classes' weight lies in [16 / total, 1] (1 = solo passes on the whole GPU), the front's in
    [(total - 16) / total, 1], and never exceeds the plain device time."""
    from paper_2509_21301_b200 import engine as E
    bits, _, _ = tiny_setup
    reqs = [make_request(TINY, (4, 4), 8, 6, 300 + i) for i in range(6)]
    e = _engine(TINY, bits)
    total = e.query_sms()[0]
    e.set_partition(mode=E.STATIC, sm_decode_dv=16, sm_decode_dp=16)
    e.kernel_stats_reset()
    e.kernel_timing(1)
    _run(e, reqs)
    e.kernel_timing(0)
    ks, sm = e.kernel_stats(), e.kernel_stats_sm()
    e.close()
    seen = 0
    for name, (ms, work, n) in ks.items():
        if n == 0:
            continue
        seen += 1
        share = sm[name] / ms
        lo = 16 / total if name.startswith("dec") or name == "lm_head" else (total - 16) / total
        assert lo - 1e-6 <= share <= 1 + 1e-6, (name, share)
    assert seen >= 4
