"""ORACLE (test infrastructure only) -- Algorithm 1 request scheduler, step by step.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may
import this.  Shares no code with the C++ controller it checks.

Follows PAPER.md Algorithm 1 and §III-D:
  * FIFO within a stage; decode has the highest priority and co-runs with the
    front stage; vision and prefill never co-run; prefill before vision.
  * decode uses in-flight batching: a request that becomes decode-ready while
    a decode iteration runs waits in Q_d and joins the next iteration
    (Merge(Q_d, req)); vision/prefill are never batched.
  * line 3-4: count pending requests, adjust the partition with Eq. 5; the
    partition is applied per forward pass.
Readings (R13-R17):
  * events of one tick: completions before arrivals, then by request id;
  * N_pend = |Q_v| + running vision + waiting/running prefill;
  * front dispatch first, then decode; decode ctx = DV (vision running),
    DP (prefill running) or SOLO (no front stage; decode takes every SM);
    a front pass gets total - s_dec, or every SM (SOLO) when no decode work
    exists at its dispatch;
  * decode batch = decode-ready requests in decode-join order, capped at B_max;
  * gen_len counts the prefill token, decode iterations = gen_len - 1.
  * SERIAL (Serial-RR, the BASELINE comparison): one pass at a time on all SMs,
    alternating a decode iteration and a front pass when both are ready.
  * PF_LIMIT (the paper's baseline): prefill-first -- one pass at a time on
    all SMs, the front stage first; "LLM decode requests are scheduled when the
    number of waiting LLM decode requests exceeds a predefined threshold (set to 5)".
    Reading (R21): decode also runs when no front work is ready.
  * MULTI_STREAM (the paper's baseline): stages co-run like Nova but every
    pass sees all SMs ("CUDA's default multi-stream scheduling policy").
  * FRONTIER: co-run like ADAPTIVE, but the decode split of a
    co-run pass is the Pareto point picked for the arrival rate estimated over the
    last lam_window arrivals (planner.frontier_pick), instead of Eq. 5.
  * CHUNK (the paper's chunked-prefill baseline: "splits a LLM prefill request into
    several chunks and batches these chunks with LLM decode requests", token budget 128).
    Reading (R26): one pass at a time on all SMs; an LLM step is a HYBRID pass
    = the next min(remaining, budget - B) prefill tokens of the request in chunked prefill
    (FIFO from the prefill queue) + the decode batch (B requests); with no prefill in progress
    a plain decode pass.  Vision encode cannot join a batch (separate weights): it runs
    as its own pass, alternating with LLM steps when both are ready, and only while no encoded
    request waits for its first chunk.  The last chunk emits the prefill token.
The same state machine drives `simulate` (virtual time, durations from curves),
which checks the worked example of SURVEY.md §8(c) c6 by hand values.
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

from .planner import adaptive_sm, arrival_rate, frontier_pick

SERIAL, STATIC, ADAPTIVE, PF_LIMIT, MULTI_STREAM, FRONTIER, CHUNK = 0, 1, 2, 3, 4, 5, 6
CTX_DV, CTX_DP, CTX_SOLO = 0, 1, 2
# event kinds (order = tie-break class: completions first)
EV_VISION_DONE, EV_PREFILL_DONE, EV_DECODE_DONE, EV_ARRIVAL, EV_HYBRID_DONE = 0, 1, 2, 3, 4
# decision kinds
D_VISION, D_PREFILL, D_DECODE, D_FINISH, D_HYBRID = 0, 1, 2, 3, 4


@dataclass
class Policy:
    mode: int = ADAPTIVE
    total_sms: int = 148
    granularity: int = 8
    sm_decode_dv: int = 72      # STATIC
    sm_decode_dp: int = 72
    sm_op_dv: int = 48          # ADAPTIVE (Eq. 5)
    sm_op_dp: int = 48
    sm_min: int = 16
    alpha_dv: float = 8.0
    alpha_dp: float = 8.0
    b_max: int = 16
    pf_threshold: int = 5       # PF_LIMIT
    frontier: list = field(default_factory=list)   # FRONTIER: (s_v, s_p, e2e, thr) Pareto points
    lam_window: int = 16        # FRONTIER: arrivals in the rate estimate
    sm_dv_floor: int = 0        # offload-aware floor of the decode split while vision co-runs (f3)
    chunk_budget: int = 128     # CHUNK: tokens per hybrid pass


@dataclass
class Req:
    rid: int
    gen_len: int
    emitted: int = 0
    join_seq: int = -1
    S: int = 1                  # LLM prefill tokens (n_v + prompt); CHUNK mode
    pre_done: int = 0           # CHUNK: prefill tokens of finished hybrid passes
    chunk_n: int = 0            # CHUNK: tokens of the hybrid pass in flight


class Alg1:
    """Algorithm 1 state machine; `tick(events)` returns the decisions taken."""

    def __init__(self, policy: Policy):
        self.p = policy
        self.reqs: dict[int, Req] = {}
        self.q_v: deque[int] = deque()
        self.prefill_wait: deque[int] = deque()
        self.vision_running: int | None = None
        self.prefill_running: int | None = None
        self.decode_running: list[int] | None = None
        self.q_d: list[int] = []            # decode-ready, kept in join order
        self.join_counter = 0
        self.last_pass = None               # SERIAL alternation
        self.arr_t: deque[int] = deque(maxlen=max(2, policy.lam_window))   # FRONTIER rate estimate
        self.chunk_req: int | None = None   # CHUNK: the request in chunked prefill
        self.log: list[tuple] = []

    # -- Eq. 5 / static split for a co-run context
    def split(self, ctx: int, n_pend: int) -> int:
        p = self.p
        if ctx == CTX_SOLO:
            return p.total_sms
        if p.mode == STATIC:
            return p.sm_decode_dv if ctx == CTX_DV else p.sm_decode_dp
        fl = p.sm_dv_floor if ctx == CTX_DV else 0
        if p.mode == FRONTIER and p.frontier:
            pt = frontier_pick(p.frontier, arrival_rate(list(self.arr_t)))
            return max(fl, pt[0] if ctx == CTX_DV else pt[1])
        if ctx == CTX_DV:
            return max(fl, adaptive_sm(p.sm_op_dv, p.sm_min, p.alpha_dv, n_pend, p.granularity))
        return max(fl, adaptive_sm(p.sm_op_dp, p.sm_min, p.alpha_dp, n_pend, p.granularity))

    def n_pend(self) -> int:
        return (len(self.q_v) + (self.vision_running is not None) + len(self.prefill_wait)
                + (self.prefill_running is not None) + (self.chunk_req is not None))

    def front_running(self) -> bool:
        return self.vision_running is not None or self.prefill_running is not None

    def busy(self) -> bool:
        return self.front_running() or self.decode_running is not None

    def _decode_ready(self, rid: int):
        r = self.reqs[rid]
        if r.join_seq < 0:
            r.join_seq = self.join_counter
            self.join_counter += 1
        self.q_d.append(rid)
        self.q_d.sort(key=lambda x: self.reqs[x].join_seq)

    def _emit(self, rid: int, out: list):
        r = self.reqs[rid]
        r.emitted += 1
        if r.emitted >= r.gen_len:
            out.append((D_FINISH, (rid,), CTX_SOLO, 0))
        else:
            self._decode_ready(rid)

    def add_request(self, rid: int, gen_len: int, S: int = 1):
        self.reqs[rid] = Req(rid, gen_len, S=S)

    def tick(self, events: list[tuple]) -> list[tuple]:
        """events: (kind, key, payload[, t_ns]) -- payload rid (or list of rids for DECODE_DONE);
        arrivals may carry their arrival time (FRONTIER's rate estimate)."""
        out: list[tuple] = []
        for ev in sorted(events, key=lambda e: (e[0] == EV_ARRIVAL, e[1], e[0])):
            kind, _, payload = ev[:3]
            if kind == EV_ARRIVAL:
                self.q_v.append(payload)
                if len(ev) > 3:
                    self.arr_t.append(ev[3])
            elif kind == EV_VISION_DONE:
                self.vision_running = None
                self.prefill_wait.append(payload)
                self.last_pass = "front"
            elif kind == EV_PREFILL_DONE:
                self.prefill_running = None
                self.last_pass = "front"
                self._emit(payload, out)
            elif kind == EV_DECODE_DONE:
                self.decode_running = None
                self.last_pass = "decode"
                for rid in payload:
                    self._emit(rid, out)
            elif kind == EV_HYBRID_DONE:      # payload[0]: the chunked prefill, payload[1:]: decode rows
                self.decode_running = None
                self.last_pass = "decode"
                r = self.reqs[payload[0]]
                r.pre_done += r.chunk_n
                if r.pre_done >= r.S:
                    self.chunk_req = None
                    self._emit(payload[0], out)
                for rid in payload[1:]:
                    self._emit(rid, out)
        npend = self.n_pend()
        if self.p.mode == CHUNK:
            self._dispatch_chunk(out)
        elif self.p.mode == SERIAL:
            self._dispatch_serial(out)
        elif self.p.mode == PF_LIMIT:
            self._dispatch_pf_limit(out)
        elif self.p.mode == MULTI_STREAM:
            if not self.front_running():
                self._dispatch_front(out, lambda c: (CTX_SOLO, 0))
            if self.decode_running is None and self.q_d:
                self._dispatch_decode(out, CTX_SOLO, self.p.total_sms)
        else:
            self._dispatch_corun(out, npend)
        self.log.extend(out)
        return out

    def _dispatch_front(self, out, ctx_fn):
        if self.prefill_wait:
            rid = self.prefill_wait.popleft()
            self.prefill_running = rid
            ctx, s = ctx_fn(CTX_DP)
            out.append((D_PREFILL, (rid,), ctx, s))
        elif self.q_v:
            rid = self.q_v.popleft()
            self.vision_running = rid
            ctx, s = ctx_fn(CTX_DV)
            out.append((D_VISION, (rid,), ctx, s))

    def _dispatch_decode(self, out, ctx, s):
        batch = self.q_d[: self.p.b_max]
        self.q_d = self.q_d[self.p.b_max:]
        self.decode_running = batch
        out.append((D_DECODE, tuple(batch), ctx, s))

    def _dispatch_corun(self, out, npend):
        if not self.front_running():
            has_decode = self.decode_running is not None or bool(self.q_d)
            self._dispatch_front(out, lambda c: (c, self.split(c, npend)) if has_decode else (CTX_SOLO, 0))
        if self.decode_running is None and self.q_d:
            if self.vision_running is not None:
                ctx = CTX_DV
            elif self.prefill_running is not None:
                ctx = CTX_DP
            else:
                ctx = CTX_SOLO
            self._dispatch_decode(out, ctx, self.split(ctx, npend))

    def _dispatch_pf_limit(self, out):
        if self.busy():
            return
        front_ready = bool(self.prefill_wait or self.q_v)
        if self.q_d and (len(self.q_d) > self.p.pf_threshold or not front_ready):
            self._dispatch_decode(out, CTX_SOLO, self.p.total_sms)
        elif front_ready:
            self._dispatch_front(out, lambda c: (CTX_SOLO, 0))

    def _dispatch_chunk(self, out):
        if self.vision_running is not None or self.decode_running is not None:
            return
        llm_ready = self.chunk_req is not None or bool(self.prefill_wait) or bool(self.q_d)
        vis_ready = bool(self.q_v) and not self.prefill_wait
        if vis_ready and (not llm_ready or self.last_pass == "decode"):
            rid = self.q_v.popleft()
            self.vision_running = rid
            out.append((D_VISION, (rid,), CTX_SOLO, 0))
            return
        if not llm_ready:
            return
        if self.chunk_req is None and self.prefill_wait:
            self.chunk_req = self.prefill_wait.popleft()
        batch = self.q_d[: self.p.b_max]
        self.q_d = self.q_d[self.p.b_max:]
        if self.chunk_req is not None:
            r = self.reqs[self.chunk_req]
            r.chunk_n = min(r.S - r.pre_done, max(1, self.p.chunk_budget - len(batch)))
            self.decode_running = [self.chunk_req] + batch
            out.append((D_HYBRID, (self.chunk_req,) + tuple(batch), CTX_SOLO, r.chunk_n))
        else:
            self.decode_running = batch
            out.append((D_DECODE, tuple(batch), CTX_SOLO, self.p.total_sms))

    def _dispatch_serial(self, out):
        if self.busy():
            return
        front_ready = bool(self.prefill_wait or self.q_v)
        dec_ready = bool(self.q_d)
        if front_ready and (not dec_ready or self.last_pass == "decode"):
            self._dispatch_front(out, lambda c: (CTX_SOLO, 0))
        elif dec_ready:
            self._dispatch_decode(out, CTX_SOLO, self.p.total_sms)


# ------------------------------------------------------------------ virtual-time simulation
@dataclass
class SimCurves:
    """Durations in ns.  Split-indexed tables give the co-run time with decode on s SMs;
    *_solo are the all-SM times.  Decode may grow linearly with batch: t*(1+beta(B-1))."""
    splits: list[int]
    t_v: list[int]
    t_p: list[int]
    t_d_dv: list[int]
    t_d_dp: list[int]
    t_v_solo: int
    t_p_solo: int
    t_d_solo: int
    beta: float = 0.0

    def idx(self, s):
        return self.splits.index(s)


@dataclass
class SimRequest:
    rid: int
    arrival_ns: int
    gen_len: int
    vis_scale: float = 1.0
    pre_scale: float = 1.0
    S: int = 1                  # LLM prefill tokens (CHUNK mode)


def simulate(policy: Policy, curves: SimCurves, requests: list[SimRequest]):
    """Run Alg. 1 in virtual integer-ns time.  Returns (decision log, token times per rid)."""
    alg = Alg1(policy)
    for r in requests:
        alg.add_request(r.rid, r.gen_len, r.S)
    byid = {r.rid: r for r in requests}
    arrivals = sorted(requests, key=lambda r: (r.arrival_ns, r.rid))
    ai = 0
    pending: list[tuple] = []     # (t_done, kind, key, payload)
    tokens: dict[int, list[int]] = {r.rid: [] for r in requests}
    done = 0
    t = 0
    while done < len(requests):
        cands = [p[0] for p in pending]
        if ai < len(arrivals):
            cands.append(arrivals[ai].arrival_ns)
        t = min(cands)
        evs = []
        for p in [p for p in pending if p[0] == t]:
            pending.remove(p)
            evs.append(p[1:])
        while ai < len(arrivals) and arrivals[ai].arrival_ns == t:
            evs.append((EV_ARRIVAL, arrivals[ai].rid, arrivals[ai].rid, arrivals[ai].arrival_ns))
            ai += 1
        for ev in evs:
            kind, payload = ev[0], ev[2]
            if kind == EV_PREFILL_DONE:
                tokens[payload].append(t)
            elif kind == EV_DECODE_DONE:
                for rid in payload:
                    tokens[rid].append(t)
            elif kind == EV_HYBRID_DONE:
                r0 = alg.reqs[payload[0]]
                if r0.pre_done + r0.chunk_n >= r0.S:     # the last chunk emits the prefill token
                    tokens[payload[0]].append(t)
                for rid in payload[1:]:
                    tokens[rid].append(t)
        for kind, rids, ctx, s in alg.tick(evs):
            if kind == D_FINISH:
                done += 1
                continue
            if kind == D_VISION:
                base = curves.t_v_solo if ctx == CTX_SOLO else curves.t_v[curves.idx(s)]
                dur = int(round(base * byid[rids[0]].vis_scale))
                pending.append((t + dur, EV_VISION_DONE, rids[0], rids[0]))
            elif kind == D_PREFILL:
                base = curves.t_p_solo if ctx == CTX_SOLO else curves.t_p[curves.idx(s)]
                dur = int(round(base * byid[rids[0]].pre_scale))
                pending.append((t + dur, EV_PREFILL_DONE, rids[0], rids[0]))
            elif kind == D_HYBRID:   # the chunk's share of the solo prefill + the decode batch
                nb = len(rids) - 1
                dd = curves.t_d_solo * (1.0 + curves.beta * (nb - 1)) if nb > 0 else 0.0
                r0 = byid[rids[0]]
                dur = int(math.floor(curves.t_p_solo * r0.pre_scale * s / r0.S + dd + 0.5))  # llround (x > 0)
                pending.append((t + dur, EV_HYBRID_DONE, min(rids), list(rids)))
            else:
                if ctx == CTX_SOLO:
                    base = curves.t_d_solo
                elif ctx == CTX_DV:
                    base = curves.t_d_dv[curves.idx(s)]
                else:
                    base = curves.t_d_dp[curves.idx(s)]
                dur = int(round(base * (1.0 + curves.beta * (len(rids) - 1))))
                pending.append((t + dur, EV_DECODE_DONE, min(rids), list(rids)))
    return alg.log, tokens
