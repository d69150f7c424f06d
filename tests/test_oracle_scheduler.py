"""Pins for oracle/scheduler.py (Algorithm 1): hand-computed worked example and
the invariants of SPEC.md S:246-251 on random traces (CPU only)."""
import random

import pytest

from oracle.scheduler import (Alg1, Policy, SimCurves, SimRequest, simulate, SERIAL, STATIC, ADAPTIVE, PF_LIMIT,
                              MULTI_STREAM,
                              D_VISION, D_PREFILL, D_DECODE, D_FINISH, CTX_DV, CTX_DP, CTX_SOLO)

MS = 1_000_000


def _curves_const(tv, tp, td, splits=(8, 16, 24)):
    n = len(splits)
    return SimCurves(list(splits), [tv] * n, [tp] * n, [td] * n, [td] * n, tv, tp, td)


def test_worked_example_nova_and_serial():
    """SURVEY.md 8(c) c6 (the fig:pipeline_parallelization scenario): t_v 10,
    t_p 4, t_d 1 ms, gen_len 3, two requests at t=0 -- values derived by hand."""
    c = _curves_const(10 * MS, 4 * MS, 1 * MS)
    reqs = [SimRequest(1, 0, 3), SimRequest(2, 0, 3)]
    pol = Policy(mode=ADAPTIVE, sm_op_dv=16, sm_op_dp=16, sm_min=8, alpha_dv=4, alpha_dp=4)
    _, tok = simulate(pol, c, reqs)
    assert tok[1] == [14 * MS, 15 * MS, 16 * MS]
    assert tok[2] == [28 * MS, 29 * MS, 30 * MS]
    # Eq. 1 closed form for r1: t_v + t_p + (gen_len - 1) t_d
    assert tok[1][-1] == (10 + 4 + 2 * 1) * MS
    _, tok = simulate(Policy(mode=SERIAL), c, reqs)
    assert tok[1] == [14 * MS, 15 * MS, 26 * MS]
    assert tok[2] == [30 * MS, 31 * MS, 32 * MS]


def test_worked_example_paper_baselines():
    """Same scenario under the paper's baselines, token times by hand.
    PF-Limit(5): r1 vision 0-10, prefill 10-14 (token 14); r1 waits in Q_d (1 <= 5) while
    r2 runs vision 14-24 and prefill 24-28 (token 28); no front work left -> decode [r1, r2]
    at 28-29 and 29-30.  With threshold 0 every waiting decode request preempts the front:
    the Serial-RR-like 14, 15, 16 / 30, 31, 32.  Multi-stream: decode of r1 co-runs with
    r2's vision on the full GPU (equal solo durations in this simulation)."""
    c = _curves_const(10 * MS, 4 * MS, 1 * MS)
    reqs = [SimRequest(1, 0, 3), SimRequest(2, 0, 3)]
    _, tok = simulate(Policy(mode=PF_LIMIT, pf_threshold=5), c, reqs)
    assert tok[1] == [14 * MS, 29 * MS, 30 * MS]
    assert tok[2] == [28 * MS, 29 * MS, 30 * MS]
    _, tok = simulate(Policy(mode=PF_LIMIT, pf_threshold=0), c, reqs)
    assert tok[1] == [14 * MS, 15 * MS, 16 * MS]
    assert tok[2] == [30 * MS, 31 * MS, 32 * MS]
    _, tok = simulate(Policy(mode=MULTI_STREAM), c, reqs)
    assert tok[1] == [14 * MS, 15 * MS, 16 * MS]
    assert tok[2] == [28 * MS, 29 * MS, 30 * MS]


def _random_trace(seed, n=40):
    rnd = random.Random(seed)
    t, out = 0, []
    for i in range(n):
        t += int(rnd.expovariate(1 / 8.0) * MS)
        out.append(SimRequest(i + 1, t, rnd.randint(1, 6), rnd.choice([1.0, 1.6]), rnd.uniform(0.8, 1.3)))
    return out


def _curves_split(splits=(8, 16, 24, 32, 40, 48)):
    tv = [int(10 * MS * 148 / (148 - s)) for s in splits]
    tp = [int(4 * MS * 148 / (148 - s)) for s in splits]
    td = [int(1 * MS * max(1.0, 24 / s)) for s in splits]
    return SimCurves(list(splits), tv, tp, td, td, 10 * MS, 4 * MS, 1 * MS, beta=0.02)


@pytest.mark.parametrize("mode", [SERIAL, STATIC, ADAPTIVE])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_alg1_invariants(mode, seed):
    reqs = _random_trace(seed)
    pol = Policy(mode=mode, sm_decode_dv=24, sm_decode_dp=16, sm_op_dv=48, sm_op_dp=40, sm_min=8,
                 alpha_dv=13.3, alpha_dp=10.7, b_max=4)
    log, tok = simulate(pol, _curves_split(), reqs)
    byid = {r.rid: r for r in reqs}
    # every request finishes exactly once with exactly gen_len tokens
    fin = [d[1][0] for d in log if d[0] == D_FINISH]
    assert sorted(fin) == sorted(byid)
    for rid, ts in tok.items():
        assert len(ts) == byid[rid].gen_len
        assert ts == sorted(ts)
    # FIFO within the vision stage (arrival order; ties by id)
    vis = [d[1][0] for d in log if d[0] == D_VISION]
    assert vis == [r.rid for r in sorted(reqs, key=lambda r: (r.arrival_ns, r.rid))]
    # decode batches respect B_max and never contain a request twice
    for d in log:
        if d[0] == D_DECODE:
            assert 1 <= len(d[1]) <= pol.b_max and len(set(d[1])) == len(d[1])
        if mode != SERIAL and d[0] in (D_VISION, D_PREFILL) and d[2] != CTX_SOLO:
            assert d[3] >= pol.sm_min or mode == STATIC


def test_vision_prefill_never_corun_and_decode_joins_next_iteration():
    """Replay the event sequence and check the running-set invariants tick by tick."""
    reqs = _random_trace(7, 30)
    pol = Policy(mode=ADAPTIVE, sm_op_dv=48, sm_op_dp=40, sm_min=8, alpha_dv=13.3, alpha_dp=10.7, b_max=16)
    alg = Alg1(pol)
    for r in reqs:
        alg.add_request(r.rid, r.gen_len)
    log, _ = simulate(pol, _curves_split(), reqs)
    # prefill of a request is dispatched before any later vision (prefill priority)
    order = [(d[0], d[1][0]) for d in log if d[0] in (D_VISION, D_PREFILL)]
    for i, (k, rid) in enumerate(order):
        if k == D_VISION and i + 1 < len(order):
            assert order[i + 1] == (D_PREFILL, rid)   # vision -> its own prefill, nothing between
    # a request's first decode iteration is the first decode dispatched after its prefill
    seen_prefill_done = set()
    for d in log:
        if d[0] == D_DECODE:
            for rid in d[1]:
                seen_prefill_done.discard(rid)
        if d[0] == D_PREFILL:
            seen_prefill_done.add(d[1][0])


def test_eq5_split_tracks_pending():
    pol = Policy(mode=ADAPTIVE, sm_op_dv=48, sm_op_dp=40, sm_min=16, alpha_dv=8, alpha_dp=8)
    a = Alg1(pol)
    assert [a.split(CTX_DV, n) for n in (0, 1, 2, 3, 4, 5)] == [48, 48, 40, 32, 24, 16]
    assert a.split(CTX_SOLO, 3) == 148
