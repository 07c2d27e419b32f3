"""Search procedures over the V-callable protocol (search.py:3-8), with the
fused device greedy.

* `model_value(params)` - V-callable backed by the device (drop-in for
  search.model_value, search.py:72-78).
* `greedy_schedule(p, V, noise, rng)` - the reference loop (search.py:90-112)
  over any V-callable; children are built without re-checking legality
  because they come from candidate_actions.
* `score_children(params, s, actions)` - V of every child of one parent
  (ts_score_children): only the new row of each child is featurized and the
  LSTM runs over only the timesteps the children differ in.  V-callables from
  `model_value` carry it and greedy_schedule uses it for each layer's
  children (bit-identical to predict_states on the children); beam_search
  keeps one predict_states batch per layer for all parents' children.
* `greedy_schedule_gpu(p, params, noise, rng)` - the fused path: per layer
  the native driver enumerates candidates, the device featurizes only the
  new row of every child, dedups identical rows, runs the exact LSTM from
  the shared prefix and returns only the winner (ts_greedy).  Same results
  as greedy_schedule(p, model_value(params)), including rng advancement.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import PipelineError
from .schedule_space import (ScheduleState, _info, candidate_actions, canonical_key, child_state,
                             initial_state)
from .value_model import MODE_EXACT, predict_states

_MASK = (1 << 64) - 1


class SearchRng:
    """splitmix64 (search.py:30-58)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + ((self.next_u64() >> 11) / float(1 << 53)) * (hi - lo)

    def randrange(self, n: int) -> int:
        return (self.next_u64() * n) >> 64

    def split(self, index: int) -> "SearchRng":
        child = SearchRng(self.state ^ (0xA5A5A5A5A5A5A5A5 + index))
        child.next_u64()
        return child


@dataclass(frozen=True)
class NoiseConfig:
    epsilon: float = 0.25

    def __post_init__(self):
        if not 0 <= self.epsilon < 1:
            raise PipelineError("epsilon must be in [0, 1)")


def model_value(params, jobs: int = 1, mode: int = MODE_EXACT):
    def fn(states):
        return predict_states(params, states, jobs=jobs, mode=mode)
    if mode == MODE_EXACT:
        if int(params.hidden) == 32:  # the fused device beam (ts_beam)
            fn.beam = lambda prefix, width: beam_search_gpu(prefix, params, width)
        fn.score_children = lambda s, actions: (
            score_children(params, s, actions) if len(actions) <= 4096
            else predict_states(params, [child_state(s, a) for a in actions], jobs=jobs, mode=mode))
    return fn


def score_children(params, s, actions, noise: NoiseConfig | None = None, rng: SearchRng | None = None,
                   device=None, best: bool = False):
    """V (exact, noise-free) of child_state(s, a) for every a in `actions`
    (legal for s, at most 4096) - or, with best=True, the index and (noisy)
    value of the argmin by (v * (1 + U(-eps, eps)), index), advancing `rng`
    by one draw per child like greedy_schedule (search.py:104-110)."""
    if not actions:
        raise PipelineError("no children to score")
    eps = float(noise.epsilon) if noise is not None else 0.0
    if eps > 0 and rng is None:
        raise PipelineError("noisy evaluation needs an rng")
    inf = _info(s.pipeline)
    ctx = _lib.context(device)
    parent = np.frombuffer(inf.records_of(s), dtype=_lib.DECISION_DTYPE)
    pos = len(s.decisions)
    kids = np.frombuffer(b"".join(inf.encode(pos, a) for a in actions), dtype=_lib.DECISION_DTYPE)
    st = ctypes.c_uint64(rng.state if rng is not None else 0)
    if best:
        bi, bv = ctypes.c_int64(), ctypes.c_double()
        with ctx.lock:  # params upload and the call that scores with them
            ctx.set_params(params)
            pid = ctx.pipeline_id(inf.desc)
            ctx.check(ctx.lib.ts_score_children(ctx.h, pid, _lib._p(parent) if len(parent) else None,
                                                len(parent), _lib._p(kids), len(kids), eps, ctypes.byref(st),
                                                None, ctypes.byref(bi), ctypes.byref(bv)))
        if rng is not None and eps > 0:
            rng.state = st.value
        return bi.value, bv.value
    out = np.empty(len(kids))
    with ctx.lock:
        ctx.set_params(params)
        pid = ctx.pipeline_id(inf.desc)
        ctx.check(ctx.lib.ts_score_children(ctx.h, pid, _lib._p(parent) if len(parent) else None,
                                            len(parent), _lib._p(kids), len(kids), 0.0, None,
                                            _lib._p(out), None, None))
    return out


def table_value(table: dict, default: float = math.inf):
    def fn(states):
        return [table.get(canonical_key(s), default) for s in states]
    return fn


def greedy_schedule(p, V, noise: NoiseConfig | None = None, rng: SearchRng | None = None):
    """Layer-by-layer argmin under V; returns (state, visited)."""
    s = initial_state(p)
    visited = 0
    while not s.is_complete:
        cands = candidate_actions(s)
        visited += len(cands)
        children = [child_state(s, a) for a in cands]
        sc = getattr(V, "score_children", None)
        vals = [float(v) for v in (sc(s, cands) if sc is not None else V(children))]
        if noise is not None and noise.epsilon > 0:
            if rng is None:
                raise PipelineError("noisy evaluation needs an rng")
            vals = [v * (1.0 + rng.uniform(-noise.epsilon, noise.epsilon)) for v in vals]
        best = min(range(len(vals)), key=lambda i: (vals[i], i))
        s = children[best]
    return s, visited


def greedy_schedule_gpu(p, params, noise: NoiseConfig | None = None,
                        rng: SearchRng | None = None, device=None, return_value=False):
    """Fused device greedy (ts_greedy); (state, visited[, V of the result])."""
    eps = float(noise.epsilon) if noise is not None else 0.0
    if eps > 0 and rng is None:
        raise PipelineError("noisy evaluation needs an rng")
    ctx = _lib.context(device)
    inf = _info(p)
    out = np.zeros(inf.T, dtype=_lib.DECISION_DTYPE)
    visited = ctypes.c_int64()
    best_v = ctypes.c_double()
    st = ctypes.c_uint64(rng.state if rng is not None else 0)
    with ctx.lock:  # params upload and the greedy that scores with them
        ctx.set_params(params)
        pid = ctx.pipeline_id(inf.desc)
        ctx.check(ctx.lib.ts_greedy(ctx.h, pid, eps, ctypes.byref(st), _lib._p(out),
                                    ctypes.byref(visited), ctypes.byref(best_v)))
    if rng is not None and eps > 0:
        rng.state = st.value
    # the chosen records are exactly the encoding of the decoded decisions
    s = ScheduleState(p, inf.decode_records(out))
    s._cache["ts_records"] = out.tobytes()
    if return_value:
        return s, visited.value, best_v.value
    return s, visited.value


def beam_search(prefix, V, width: int = 8):
    """Beam over completions of `prefix` (search.py:115-133).  A model_value
    V-callable carries the fused device beam (ts_beam: one device pass per
    layer for all parents' children, no per-child host states); any other V
    goes through the generic loop below."""
    if width < 1:
        raise PipelineError("beam width must be >= 1")
    fused = getattr(V, "beam", None)
    if fused is not None:
        return fused(prefix, width)
    frontier = [prefix]
    while not frontier[0].is_complete:
        # one device batch per layer for all parents' children (per-parent
        # score_children calls would cost one round trip per beam entry)
        children = []
        for s in frontier:
            children.extend(child_state(s, a) for a in candidate_actions(s))
        vals = V(children)
        ranked = sorted(range(len(children)), key=lambda i: (float(vals[i]), i))
        frontier = [children[i] for i in ranked[:width]]
    vals = V(frontier)
    best = min(range(len(frontier)), key=lambda i: (float(vals[i]), i))
    return frontier[best]


def beam_search_gpu(prefix, params, width: int = 8, device=None, return_value=False):
    """Fused device beam_search(prefix, model_value(params), width)
    (ts_beam); the returned state's decisions are the prefix's followed by
    the completion.  (state[, V of the state])."""
    if width < 1:
        raise PipelineError("beam width must be >= 1")
    p = prefix.pipeline
    inf = _info(p)
    ctx = _lib.context(device)
    pre = np.frombuffer(inf.records_of(prefix), dtype=_lib.DECISION_DTYPE)
    out = np.zeros(inf.T, dtype=_lib.DECISION_DTYPE)
    visited = ctypes.c_int64()
    best_v = ctypes.c_double()
    with ctx.lock:  # params upload and the beam that scores with them
        ctx.set_params(params)
        pid = ctx.pipeline_id(inf.desc)
        ctx.check(ctx.lib.ts_beam(ctx.h, pid, _lib._p(pre) if len(pre) else None, len(pre), int(width),
                                  _lib._p(out), ctypes.byref(visited), ctypes.byref(best_v)))
    d = len(prefix.decisions)
    s = ScheduleState(p, tuple(prefix.decisions) + inf.decode_records(out[d:], d))
    s._cache["ts_records"] = out.tobytes()
    if return_value:
        return s, best_v.value
    return s


def random_schedule(p, rng: SearchRng):
    s = initial_state(p)
    while not s.is_complete:
        cands = candidate_actions(s)
        s = child_state(s, cands[rng.randrange(len(cands))])
    return s
