"""Host mirror of the reference pipeline IR (pipeline_ir.py) plus the flat
device descriptor.

Only what the scoring path needs is mirrored: the data model with the
reference's attribute names (so the reference's own `Pipeline` objects can be
passed in unchanged - everything here is duck-typed), the text format,
topological / schedule order, and `descriptor()`, which lowers a pipeline to
the int64 words `ts_pipeline_upload` consumes (layout in DESIGN.md).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import CycleError, ParseError, PipelineError, UnknownStageError

STAGE_ELEM_SIZE = 4  # pipeline_ir.py:17
DESC_MAGIC = 0x54534231
DESC_STAGE_WORDS = 48
MAX_PURE, MAX_RED, MAX_LOOPS = 4, 4, 8
_I63 = (1 << 63) - 1


@dataclass(frozen=True)
class AccessMap:
    consumer_dim: int | None
    stride: int
    window: int


@dataclass(frozen=True)
class InputEdge:
    producer: str
    access: tuple


@dataclass(frozen=True)
class Stage:
    name: str
    dims: tuple
    reduction_dims: tuple
    flops_per_point: int
    inputs: tuple
    output: bool = False

    @property
    def all_dims(self):
        return self.dims + self.reduction_dims

    @property
    def pure_extents(self):
        return tuple(e for _, e in self.dims)

    @property
    def reduction_extents(self):
        return tuple(e for _, e in self.reduction_dims)

    @property
    def domain_points(self):
        return math.prod(self.pure_extents) * math.prod(self.reduction_extents)


@dataclass(frozen=True)
class ExternalBuffer:
    name: str
    dims: tuple
    element_size: int


@dataclass(frozen=True)
class Pipeline:
    name: str
    buffers: tuple
    stages: tuple
    _cache: dict = field(default_factory=dict, compare=False, repr=False, hash=False)

    def __hash__(self):
        h = self._cache.get("hash")
        if h is None:
            h = self._cache["hash"] = hash((self.name, self.buffers, self.stages))
        return h

    def stage(self, name):
        for s in self.stages:
            if s.name == name:
                return s
        raise UnknownStageError(f"unknown stage {name!r}")


def _stage_index(p) -> dict:
    return {s.name: s for s in p.stages}


def topological_order(p) -> list:
    """Producers before consumers, ties by declaration order (pipeline_ir.py:179-204)."""
    names = [s.name for s in p.stages]
    known = set(names)
    deps = {s.name: {e.producer for e in s.inputs if e.producer in known} for s in p.stages}
    order, placed = [], set()
    while len(order) < len(names):
        # one declaration-order pass places every ready stage, re-checking
        # readiness as earlier stages of the same pass get placed
        progressed = False
        for n in names:
            if n not in placed and deps[n] <= placed:
                order.append(n)
                placed.add(n)
                progressed = True
        if not progressed:
            raise CycleError(f"cycle among stages {[n for n in names if n not in placed]}")
    return order


def schedule_order(p) -> list:
    """Consumers first (pipeline_ir.py:207-213)."""
    return topological_order(p)[::-1]


def consumers_of(p, name) -> tuple:
    return tuple(s.name for s in p.stages if any(e.producer == name for e in s.inputs))


def consumer_map(p) -> dict:
    """consumers_of for every stage in one pass (name -> consumers in stage order)."""
    out = {s.name: [] for s in p.stages}
    for s in p.stages:
        seen = set()
        for e in s.inputs:
            if e.producer in out and e.producer not in seen:
                seen.add(e.producer)
                out[e.producer].append(s.name)
    return {k: tuple(v) for k, v in out.items()}


# ------------------------------------------------------------- text format
def _dim_list(text, lineno):
    out = []
    for part in text.split(","):
        bits = part.split(":")
        if len(bits) != 2:
            raise ParseError(f"bad dim spec {part!r}", lineno)
        try:
            out.append((bits[0].strip(), int(bits[1])))
        except ValueError:
            raise ParseError(f"bad dim spec {part!r}", lineno) from None
    return tuple(out)


def _map_clause(text, dim_index, lineno):
    text = text.strip()
    ref, star, rest = text.partition("*")
    s_txt, plus, w_txt = rest.partition("+")
    try:
        if not star or not plus:
            raise ValueError
        stride, window = int(s_txt), int(w_txt)
    except ValueError:
        raise ParseError(f"bad map clause {text!r}", lineno) from None
    ref = ref.strip()
    if ref == "_":
        return AccessMap(None, stride, window)
    if ref not in dim_index:
        raise ParseError(f"unknown consumer dim {ref!r} in map clause", lineno)
    return AccessMap(dim_index[ref], stride, window)


def parse_pipeline(text: str) -> Pipeline:
    """Line-oriented pipeline spec (pipeline_ir.py:347-352 grammar)."""
    name = None
    buffers, stages, known = [], [], set()
    cur = None

    def close():
        if cur is not None:
            stages.append(Stage(cur[0], cur[1], cur[2], cur[3], tuple(cur[4]), cur[5]))

    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        toks = line.split()
        kw = toks[0]
        if kw == "pipeline":
            if len(toks) != 2:
                raise ParseError("expected: pipeline <name>", lineno)
            name = toks[1]
        elif kw == "buffer":
            if len(toks) != 6 or toks[2] != "dims" or toks[4] != "elem":
                raise ParseError("expected: buffer <name> dims <e1>x... elem <bytes>", lineno)
            if toks[1] in known:
                raise ParseError(f"duplicate name {toks[1]!r}", lineno)
            try:
                buffers.append(ExternalBuffer(toks[1], tuple(int(x) for x in toks[3].split("x")),
                                              int(toks[5])))
            except ValueError:
                raise ParseError("bad buffer dims/elem", lineno) from None
            known.add(toks[1])
        elif kw == "stage":
            close()
            cur = None
            if len(toks) < 5 or toks[2] != "dims":
                raise ParseError("expected: stage <name> dims <d>:<e>,... [reduce ...] "
                                 "flops <k> [output]", lineno)
            if toks[1] in known:
                raise ParseError(f"duplicate name {toks[1]!r}", lineno)
            rest = toks[4:]
            red = ()
            if rest and rest[0] == "reduce":
                if len(rest) < 2:
                    raise ParseError("reduce needs a dim list", lineno)
                red = _dim_list(rest[1], lineno)
                rest = rest[2:]
            if len(rest) < 2 or rest[0] != "flops":
                raise ParseError("expected flops <k>", lineno)
            try:
                flops = int(rest[1])
            except ValueError:
                raise ParseError(f"bad flops count {rest[1]!r}", lineno) from None
            tail = rest[2:]
            if tail not in ([], ["output"]):
                raise ParseError(f"unexpected tokens {tail}", lineno)
            cur = [toks[1], _dim_list(toks[3], lineno), red, flops, [], tail == ["output"]]
            known.add(toks[1])
        elif kw == "in":
            if cur is None:
                raise ParseError("'in' line outside a stage", lineno)
            if len(toks) < 4 or toks[2] != "map":
                raise ParseError("expected: in <producer> map <clauses>", lineno)
            if toks[1] not in known:
                raise ParseError(f"unknown reference {toks[1]!r}", lineno)
            dim_index = {d: i for i, (d, _) in enumerate(cur[1] + cur[2])}
            clauses = " ".join(toks[3:]).split(",")
            cur[4].append(InputEdge(toks[1], tuple(_map_clause(c, dim_index, lineno)
                                                   for c in clauses)))
        else:
            raise ParseError(f"unknown directive {kw!r}", lineno)
    close()
    if name is None:
        raise ParseError("missing 'pipeline <name>' line")
    return Pipeline(name, tuple(buffers), tuple(stages))


# ------------------------------------------------------------- descriptor
def _producer_info(p, name):
    st = _stage_index(p)
    if name in st:
        return st[name].pure_extents, STAGE_ELEM_SIZE
    for b in p.buffers:
        if b.name == name:
            return tuple(b.dims), b.element_size
    raise PipelineError(f"unknown producer {name!r}")


def _footprint_size(edge, extents):
    """Size of the access-map image of the full consumer domain (pipeline_ir.py:216-230)."""
    size = 1
    for am in edge.access:
        if am.consumer_dim is None:
            size *= am.window
        else:
            size *= am.stride * (extents[am.consumer_dim] - 1) + am.window
    return size


def _checked(v, what):
    if not 0 <= v <= _I63:
        raise PipelineError(f"{what} = {v} outside the 63-bit descriptor envelope")
    return v


def descriptor(p) -> np.ndarray:
    """Lower a (duck-typed) pipeline to the `ts_pipeline_upload` word array.

    Stages are indexed by topological position (the feature row).  Besides
    the static nest inputs it carries the schedule-invariant integers behind
    the intrinsic features (pipeline_ir.py:241-252; featurizer.py:44-65) and a
    static liveness allocation of nest slots: a stage's nest is kept only
    while a producer whose sole consumer it is remains unscheduled.
    """
    hit = _DESC_CACHE.get(p)
    if hit is not None:
        return hit
    topo = topological_order(p)
    T = len(topo)
    pos = {n: i for i, n in enumerate(topo)}
    st = _stage_index(p)
    sole = {}
    cmap = consumer_map(p)
    for n in topo:
        cons = cmap[n]
        sole[n] = cons[0] if len(cons) == 1 else None
    # slot allocation over schedule indices (sched(s) = T-1-pos(s))
    live_end = {}
    for n in topo:
        c = sole[n]
        if c is not None:
            live_end[c] = max(live_end.get(c, -1), T - 1 - pos[n])
    slots, free_at = {}, []  # free_at[k] = schedule index after which slot k is free
    for c in sorted(live_end, key=lambda n: T - 1 - pos[n]):
        start = T - 1 - pos[c]
        for k, end in enumerate(free_at):
            if end < start:
                slots[c] = k
                free_at[k] = live_end[c]
                break
        else:
            slots[c] = len(free_at)
            free_at.append(live_end[c])
    words = [DESC_MAGIC, T, len(free_at), 0]
    for n in topo:
        s = st[n]
        n_pure, n_red = len(s.dims), len(s.reduction_dims)
        if not 1 <= n_pure <= MAX_PURE or n_red > MAX_RED:
            raise PipelineError(f"stage {n}: {n_pure} pure / {n_red} reduction dims outside "
                                f"the 4/4 envelope")
        ext = [e for _, e in s.dims] + [e for _, e in s.reduction_dims]
        pure_points = math.prod(ext[:n_pure])
        red_points = math.prod(ext[n_pure:])
        points = pure_points * red_points
        in_bytes = 0
        ov = Fraction(0)
        ov_pair = (0, 1)
        for e in s.inputs:
            _, elem = _producer_info(p, e.producer)
            in_bytes += _footprint_size(e, ext) * elem
            for am in e.access:
                r = Fraction(am.window, max(1, am.stride))
                if r > ov:
                    ov, ov_pair = r, (am.window, am.stride)
        out_bytes = pure_points * STAGE_ELEM_SIZE
        c = sole[n]
        cedges = [e for e in st[c].inputs if e.producer == n] if c is not None else []
        if len(cedges) > 2:
            raise PipelineError(f"stage {n}: more than 2 parallel edges from its consumer")
        cdim = [[-1] * 4 for _ in range(2)]
        cstride = [[0] * 4 for _ in range(2)]
        cwin = [[0] * 4 for _ in range(2)]
        for ei, e in enumerate(cedges):
            if len(e.access) != n_pure:
                raise PipelineError(f"edge {c} <- {n}: access arity")
            for k, am in enumerate(e.access):
                cdim[ei][k] = -1 if am.consumer_dim is None else am.consumer_dim
                cstride[ei][k] = am.stride
                cwin[ei][k] = am.window
        w = [n_pure, n_red] + ext + [0] * (8 - len(ext))
        w += [_checked(pure_points, "pure points"), _checked(red_points, "reduction points"),
              _checked(points, "domain points"), _checked(points, "points"),
              _checked(points * s.flops_per_point, "flops"), _checked(in_bytes, "input bytes"),
              _checked(out_bytes, "output bytes")]
        if in_bytes + out_bytes + 1 > _I63:
            raise PipelineError(f"stage {n}: byte counts outside the envelope")
        w += [len(s.inputs), ov_pair[0], ov_pair[1], pos[c] if c is not None else -1, len(cedges)]
        w += sum(cdim, []) + sum(cstride, []) + sum(cwin, [])
        w += [slots.get(n, -1), min(2, n_pure)]
        assert len(w) == DESC_STAGE_WORDS
        words += w
    arr = np.array(words, dtype=np.int64)
    arr.setflags(write=False)
    _DESC_CACHE[p] = arr
    return arr


_DESC_CACHE: dict = {}
