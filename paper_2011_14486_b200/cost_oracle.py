"""The analytical cost oracle on the B200 (cost_oracle.py).

`benchmark(s, m)` / `benchmark_states(states, m)` evaluate the reference's
deterministic fixed-point cost (cost_oracle.py:313-357) on the device with
256-bit integers (totals reach 2^145), so simulated-cost training targets
and the learner's stitched-schedule costs no longer need the Python oracle.
Only `total_millis` is produced (the per-stage breakdown of the CLI's
`bench` command is out of scope).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import PipelineError
from .pipeline_ir import STAGE_ELEM_SIZE, topological_order
from .schedule_space import encode_states

MAX_IN, MAX_MAPS = 4, 6
WORDS_PER_IN = 3 + 3 * MAX_MAPS
WORDS_PER_STAGE = 2 + MAX_IN * WORDS_PER_IN


@dataclass(frozen=True)
class MachineModel:
    """cost_oracle.py:172-193."""

    flop_cost: int = 1
    mem_byte_cost: int = 8
    cache_byte_cost: int = 1
    cache_size: int = 32768
    cores: int = 4
    task_overhead: int = 1000
    vec_widths: tuple = (1, 4, 8, 16)

    def __post_init__(self):
        if min(self.flop_cost, self.mem_byte_cost, self.cache_byte_cost, self.cache_size,
               self.cores, self.task_overhead) < 1:
            raise PipelineError("machine model parameters must be positive")
        if self.cache_byte_cost > self.mem_byte_cost:
            raise PipelineError("cache_byte_cost must not exceed mem_byte_cost")

    def words(self) -> np.ndarray:
        return np.array([self.flop_cost, self.mem_byte_cost, self.cache_byte_cost,
                         self.cache_size, self.cores, self.task_overhead], dtype=np.uint64)


def format_millis(m: int) -> str:
    return f"{m // 1000}.{m % 1000:03d}"


@dataclass(frozen=True)
class Cost:
    total_millis: int

    def __lt__(self, other):
        return self.total_millis < other.total_millis

    def __str__(self):
        return format_millis(self.total_millis)


_DESC: dict = {}


def cost_descriptor(p) -> np.ndarray:
    """Per-stage input edges in topological order (the cost-term inputs)."""
    hit = _DESC.get(p)
    if hit is not None:
        return hit
    topo = topological_order(p)
    pos = {n: i for i, n in enumerate(topo)}
    by = {s.name: s for s in p.stages}
    bufs = {b.name: b for b in p.buffers}
    words = []
    for n in topo:
        s = by[n]
        if len(s.inputs) > MAX_IN:
            raise PipelineError(f"stage {n}: more than {MAX_IN} inputs")
        w = [s.flops_per_point, len(s.inputs)]
        for e in list(s.inputs) + [None] * (MAX_IN - len(s.inputs)):
            if e is None:
                w += [0] * WORDS_PER_IN
                continue
            if len(e.access) > MAX_MAPS:
                raise PipelineError(f"stage {n}: producer {e.producer} has > {MAX_MAPS} dims")
            elem = STAGE_ELEM_SIZE if e.producer in by else bufs[e.producer].element_size
            w += [pos.get(e.producer, -1), elem, len(e.access)]
            for k in range(MAX_MAPS):
                if k < len(e.access):
                    am = e.access[k]
                    w += [-1 if am.consumer_dim is None else am.consumer_dim, am.stride, am.window]
                else:
                    w += [0, 0, 0]
        words += w
    arr = np.array(words, dtype=np.int64)
    _DESC[p] = arr
    return arr


def benchmark_states(states, m: MachineModel | None = None, device=None) -> list:
    """total_millis (Python ints) of complete schedules, on the device."""
    m = m or MachineModel()
    out = [None] * len(states)
    if not states:
        return out
    for s in states:
        if len(s.decisions) != len(s.pipeline.stages):
            raise PipelineError(f"schedule covers {len(s.decisions)}/{len(s.pipeline.stages)} stages")
    ctx = _lib.context(device)
    mw = m.words()
    for inf, idxs, recs, offsets in encode_states(states):
        pid = ctx.pipeline_id(inf.desc)
        cd = cost_descriptor(inf.p)
        limbs = np.empty((len(idxs), 4), dtype=np.uint64)
        with ctx.lock:
            ctx.check(ctx.lib.ts_benchmark(ctx.h, pid, _lib._p(cd), cd.size, _lib._p(mw),
                                           _lib._p(recs), _lib._p(offsets), len(idxs),
                                           _lib._p(limbs)))
        for j, i in enumerate(idxs):
            out[i] = sum(int(limbs[j, k]) << (64 * k) for k in range(4))
    return out


def benchmark(s, m: MachineModel | None = None) -> Cost:
    return Cost(benchmark_states([s], m)[0])


def machine_with(m: MachineModel, **kw) -> MachineModel:
    return replace(m, **kw)
