"""Host mirror of the reference MDP states/actions (schedule_space.py) and
the 16-byte decision records the device consumes.

`LayerSchedule` / `ScheduleState` keep the reference's field names and
rendering, so states built by the reference package itself can be scored
unchanged (everything below is duck-typed on `.pipeline` / `.decisions`).
Candidate enumeration and legality run in the native library
(`ts_candidates`, `ts_check_action`); Python only encodes and decodes.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import IllegalActionError, PipelineError
from .pipeline_ir import consumer_map, consumers_of, descriptor, schedule_order, topological_order

SPLIT_FACTORS = (8, 32)  # schedule_space.py:28-30
VEC_WIDTHS = (1, 8)
MAX_COMPUTE_AT_LEVELS = 3
FLAG_PARALLEL, FLAG_STORE_AT = 1, 2
_REC = struct.Struct("<4B8B3Bb")  # ts_decision: split[4], order[8], n_loops, vec, flags, anchor


@dataclass(frozen=True)
class LayerSchedule:
    stage: str
    splits: tuple
    order: tuple
    vectorize_width: int = 1
    parallel: bool = False
    compute_at: tuple | None = None
    store_at: tuple | None = None

    def render(self) -> str:
        splits = ",".join(f"{d}:{f}" for d, f in self.splits) or "-"
        at = "root" if self.compute_at is None else f"{self.compute_at[0]}@{self.compute_at[1]}"
        st = "root" if self.store_at is None else f"{self.store_at[0]}@{self.store_at[1]}"
        return (f"{self.stage} split={splits} order={','.join(self.order)} "
                f"vec={self.vectorize_width} par={int(self.parallel)} at={at} store={st}")


def parse_layer_schedule(text: str) -> LayerSchedule:
    toks = text.split()
    if len(toks) != 7:
        raise PipelineError(f"bad schedule line: {text!r}")
    kv = {}
    for tok in toks[1:]:
        k, eq, v = tok.partition("=")
        if not eq:
            raise PipelineError(f"bad schedule token {tok!r}")
        kv[k] = v

    def site(v):
        if v == "root":
            return None
        c, lvl = v.split("@")
        return (c, int(lvl))

    try:
        splits = () if kv["split"] == "-" else tuple(
            (a, int(b)) for a, b in (x.split(":") for x in kv["split"].split(",")))
        return LayerSchedule(toks[0], splits, tuple(kv["order"].split(",")), int(kv["vec"]),
                             bool(int(kv["par"])), site(kv["at"]), site(kv["store"]))
    except (KeyError, ValueError) as e:
        raise PipelineError(f"bad schedule line {text!r}: {e}") from None


@dataclass(frozen=True)
class ScheduleState:
    pipeline: object
    decisions: tuple = ()
    _cache: dict = field(default_factory=dict, compare=False, repr=False, hash=False)

    def __hash__(self):
        return hash((self.pipeline.name, self.decisions))

    @property
    def scheduled_count(self) -> int:
        return len(self.decisions)

    @property
    def order(self):
        return _info(self.pipeline).sched

    @property
    def is_complete(self) -> bool:
        return len(self.decisions) == len(self.pipeline.stages)

    @property
    def next_stage_name(self) -> str:
        return self.order[len(self.decisions)]


def initial_state(p) -> ScheduleState:
    if not p.stages:
        raise PipelineError("pipeline has no stages")
    return ScheduleState(p)


def canonical_key(s) -> str:
    return s.pipeline.name + "/" + ";".join(d.render() for d in s.decisions)


def write_schedule(s) -> str:
    return "\n".join(d.render() for d in s.decisions) + "\n"


# ---------------------------------------------------------------- records
class _PipelineInfo:
    """Per-pipeline encoding tables (cached by pipeline object)."""

    def __init__(self, p):
        self.p = p
        self.desc = descriptor(p)
        self.topo = topological_order(p)
        self.sched = self.topo[::-1]
        self.T = len(self.topo)
        by_name = {s.name: s for s in p.stages}
        self.stages = [by_name[n] for n in self.sched]
        self.sole = []
        self.loop_ids = []    # per schedule index: (split-set) -> {loop name: id}
        cmap = consumer_map(p)
        for st in self.stages:
            cons = cmap[st.name]
            self.sole.append(cons[0] if len(cons) == 1 else None)
        # the native encoder's stage table (csrc/hostenc.c): per schedule
        # index (name, pure dims, reduction dims, sole consumer), None where
        # two loop names could coincide (those stages take the Python path)
        stab = []
        for st, sole in zip(self.stages, self.sole):
            pure = tuple(n for n, _ in st.dims)
            red = tuple(n for n, _ in st.reduction_dims)
            names = [*pure, *(n + "o" for n in pure), *(n + "i" for n in pure), *red]
            ok = (len(set(names)) == len(names) and 1 <= len(pure) <= 4 and len(red) <= 4
                  and all(isinstance(n, str) for n in names))
            stab.append((st.name, pure, red, sole) if ok else None)
        self.stab = tuple(stab)
        self.enc_cache = {}   # id(decision) -> (decision, bytes, schedule index)
        # (schedule index, decision) -> bytes: decisions are frozen dataclasses,
        # so equal decisions built by any caller (a foreign search's own
        # objects) encode once; bounded by the distinct actions per stage
        self.val_cache = {}
        self.dec_cache = {}   # (schedule index, record bytes) -> decision

    def loop_table(self, st, split):
        table = {}
        for k, (d, _) in enumerate(st.dims):
            if d in split:
                table[d + "o"] = 2 * k
                table[d + "i"] = 2 * k + 1
            else:
                table[d] = 2 * k
        for r, (d, _) in enumerate(st.reduction_dims):
            table[d] = 8 + r
        return table

    def encode(self, idx: int, d) -> bytes:
        hit = self.enc_cache.get(id(d))
        if hit is not None and hit[0] is d and hit[2] == idx:  # a record is only valid at its stage
            return hit[1]
        try:
            key = (idx, d.stage, d.splits, d.order, d.vectorize_width, d.parallel, d.compute_at,
                   d.store_at)
            b = self.val_cache.get(key)
        except (TypeError, AttributeError):  # an unhashable or incomplete decision-like object
            key, b = None, None
        if b is None:
            b = self._encode_fields(idx, d)
            if key is not None and len(self.val_cache) < (1 << 20):
                self.val_cache[key] = b
        if len(self.enc_cache) >= (1 << 20):  # bounded: foreign callers bring new objects
            self.enc_cache.clear()
        self.enc_cache[id(d)] = (d, b, idx)
        return b

    def _encode_fields(self, idx: int, d) -> bytes:
        """The 16-byte ts_decision of decision d at schedule index idx."""
        st = self.stages[idx]
        if d.stage != st.name:
            raise IllegalActionError(
                f"expected a decision for stage {st.name!r}, got {d.stage!r}")
        pure = [n for n, _ in st.dims]
        split = {}
        sp = [0, 0, 0, 0]
        for dim, f in d.splits:
            if dim in split:
                raise IllegalActionError(f"{st.name}: dim {dim} split twice")
            if dim not in pure:
                raise IllegalActionError(f"{st.name}: cannot split non-pure dim {dim}")
            if f < 2:
                raise IllegalActionError(f"{st.name}: split factor {f} < 2")
            if f > 255:
                raise PipelineError(f"{st.name}: split factor {f} outside the record envelope")
            split[dim] = f
            sp[pure.index(dim)] = f
        table = self.loop_table(st, split)
        if sorted(d.order) != sorted(table) or len(d.order) > 8:
            raise IllegalActionError(
                f"{st.name}: order {d.order} is not a permutation of loops {sorted(table)}")
        order = [table[name] for name in d.order] + [0xFF] * (8 - len(d.order))
        if not 1 <= d.vectorize_width <= 255:
            raise IllegalActionError(f"{st.name}: bad vectorize width {d.vectorize_width}")
        flags = FLAG_PARALLEL if d.parallel else 0
        if d.compute_at is None:
            anchor = -1
            if d.store_at is not None:
                raise IllegalActionError(f"{st.name}: store_at must be Root or the compute_at site")
        else:
            cname, lvl = d.compute_at
            if self.sole[idx] != cname:
                cons = list(consumers_of(self.p, st.name))
                raise IllegalActionError(
                    f"{st.name}: compute_at target must be the sole consumer (consumers: {cons})")
            if not 0 <= lvl < 8:
                raise IllegalActionError(f"{st.name}: loop level {lvl} does not exist in {cname}'s nest")
            anchor = lvl
            if d.store_at is not None:
                if d.store_at != d.compute_at:
                    raise IllegalActionError(
                        f"{st.name}: store_at must be Root or the compute_at site")
                flags |= FLAG_STORE_AT
        return _REC.pack(*sp, *order, len(d.order), d.vectorize_width, flags, anchor)

    def decode(self, idx: int, rec) -> LayerSchedule:
        """The decision a 16-byte record encodes at schedule index idx."""
        return self.decode_bytes(idx, rec.tobytes())

    def decode_bytes(self, idx: int, b: bytes) -> LayerSchedule:
        # decisions are frozen dataclasses: one object per (index, record),
        # shared by every caller (greedy/beam results, candidate_actions)
        key = (idx, b)
        d = self.dec_cache.get(key)
        if d is not None:
            return d
        f = _REC.unpack(b)
        st = self.stages[idx]
        split = {}
        splits = []
        for k, (dname, _) in enumerate(st.dims):
            if f[k]:
                split[dname] = f[k]
                splits.append((dname, f[k]))
        inv = {v: k for k, v in self.loop_table(st, split).items()}
        order = tuple(inv[x] for x in f[4:4 + f[12]])
        vec, flags, anchor = f[13], f[14], f[15]
        at = None if anchor < 0 else (self.sole[idx], anchor)
        store = at if (flags & FLAG_STORE_AT) else None
        d = LayerSchedule(st.name, tuple(splits), order, vec, bool(flags & FLAG_PARALLEL), at, store)
        if len(self.dec_cache) < (1 << 20):
            self.dec_cache[key] = d
        return d

    def decode_records(self, recs, start: int = 0) -> tuple:
        """Decisions of consecutive schedule indices start.. from a record array."""
        b = np.ascontiguousarray(recs).tobytes()
        return tuple(self.decode_bytes(start + i, b[16 * i:16 * i + 16]) for i in range(len(b) // 16))

    def records_of(self, s) -> bytes:
        cached = getattr(s, "_cache", None)
        if isinstance(cached, dict):
            hit = cached.get("ts_records")
            if hit is not None:
                return hit
        out = b"".join(self.encode(i, d) for i, d in enumerate(s.decisions))
        if isinstance(cached, dict):
            cached["ts_records"] = out
        return out


try:  # the native host encoder (built in-tree by build.py)
    from . import _hostenc
except ImportError:  # not built: the Python path below (host-only, same records)
    _hostenc = None

_INFO: dict = {}
_INFO_ID: dict = {}  # id(pipeline) -> (pipeline, info): no hashing of the object


def _info(p) -> _PipelineInfo:
    # identity first: hashing a Pipeline (a frozen dataclass in the
    # reference) walks every stage, ~0.3 ms for VGG-16
    hit = _INFO_ID.get(id(p))
    if hit is not None and hit[0] is p:
        return hit[1]
    cache = getattr(p, "_cache", None)
    inf = cache.get("ts_info") if isinstance(cache, dict) else None
    if inf is None:
        inf = _INFO.get(p)
        if inf is None:
            inf = _INFO[p] = _PipelineInfo(p)
        if isinstance(cache, dict):
            cache["ts_info"] = inf
    if len(_INFO_ID) > 4096:
        _INFO_ID.clear()
    _INFO_ID[id(p)] = (p, inf)  # the strong reference keeps the id valid
    return inf


def encode_states(states):
    """Group states by pipeline -> [(pipeline_info, indices, records, offsets)]."""
    groups = {}
    for i, s in enumerate(states):
        p = s.pipeline
        g = groups.get(id(p))
        if g is None:
            g = groups[id(p)] = (p, [])
        g[1].append(i)
    out = []
    for p, idxs in groups.values():
        inf = _info(p)
        if _hostenc is not None:  # native: one C call per group (csrc/hostenc.c)
            try:
                rb, ob = _hostenc.encode_group(states, idxs, inf.T, inf.encode, inf.val_cache, inf.stab)
            except ValueError as e:
                raise IllegalActionError(str(e)) from None
            recs = np.frombuffer(rb, dtype=_lib.DECISION_DTYPE)
            offsets = np.frombuffer(ob, dtype=np.int64)
            out.append((inf, idxs, recs, offsets))
            continue
        chunks = [inf.records_of(states[i]) for i in idxs]
        lens = np.fromiter((len(c) // 16 for c in chunks), dtype=np.int64, count=len(chunks))
        if np.any(lens > inf.T):
            raise IllegalActionError("state has more decisions than stages")
        offsets = np.zeros(len(chunks) + 1, dtype=np.int64)
        np.cumsum(lens, out=offsets[1:])
        recs = np.frombuffer(b"".join(chunks), dtype=_lib.DECISION_DTYPE)
        out.append((inf, idxs, recs, offsets))
    return out


# ------------------------------------------------------- action codes
# 16-bit codes of decisions in candidate_actions' space (layout:
# include/tensched_b200.h, ts_score_states_coded).
_SPLIT_CODE = np.full(256, 255, dtype=np.uint8)
_SPLIT_CODE[[0, 8, 32]] = [0, 1, 2]


def _order_variants(st, split_mask):
    """The four (placement, swap) orders of _order_options (schedule_space.py
    :361-376) as loop-id bytes packed little-endian into a u64, for a stage
    whose splittable dims are split per `split_mask` (bit 0: dims[-2:][0])."""
    n_pure, n_red = len(st.dims), len(st.reduction_dims)
    first = n_pure - 2 if n_pure >= 2 else 0
    pure = []
    for k in range(n_pure):
        pure.append(2 * k)
        if first <= k < first + 2 and (split_mask >> (k - first)) & 1:
            pure.append(2 * k + 1)
    red = [8 + r for r in range(n_red)]
    out = []
    for outer in (0, 1):
        for swap in (0, 1):
            seq = (red + pure) if outer else (pure + red)
            if swap and len(seq) >= 2:
                seq = seq[:-2] + [seq[-1], seq[-2]]
            if len(seq) > 8:
                out.append(None)
                continue
            b = bytes(seq) + b"\xff" * (8 - len(seq))
            out.append(int.from_bytes(b, "little"))
    return out


def action_codes(inf, recs, offsets):
    """Decision records (schedule order per state) -> u16 action codes, or None
    when some decision lies outside candidate_actions' space."""
    n = len(recs)
    if n == 0:
        return np.zeros(0, dtype=np.uint16)
    depths = np.diff(offsets)
    pos = np.arange(n, dtype=np.int64) - np.repeat(offsets[:-1], depths)
    n_pure = np.array([len(st.dims) for st in inf.stages], dtype=np.int64)[pos]
    first = np.where(n_pure >= 2, n_pure - 2, 0)
    split = recs["split"].astype(np.int64)
    sc = _SPLIT_CODE[recs["split"]]
    rows = np.arange(n)
    s0 = sc[rows, first]
    s1 = np.where(n_pure >= 2, sc[rows, np.minimum(first + 1, 3)], 0)
    # splits only on the splittable dims, by SPLIT_FACTORS
    kk = np.arange(4)[None, :]
    other = (kk != first[:, None]) & ((kk != first[:, None] + 1) | (n_pure[:, None] < 2))
    if np.any(split[other] != 0) or np.any(s0 == 255) or np.any(s1 == 255):
        return None
    anchor = recs["anchor"].astype(np.int64)
    vec = recs["vec"].astype(np.int64)
    flags = recs["flags"].astype(np.int64)
    if np.any((anchor < -1) | (anchor > 2)) or np.any((vec != 1) & (vec != 8)) or np.any(flags > 3):
        return None
    order = np.ascontiguousarray(recs["order"]).view("<u8").ravel()
    mask = (s0 != 0).astype(np.int64) | ((s1 != 0).astype(np.int64) << 1)
    key = pos * 4 + mask
    ob = np.full(n, -1, dtype=np.int64)
    for k in np.unique(key):
        sel = key == k
        st = inf.stages[int(k) // 4]
        got = order[sel]
        bits = np.full(got.shape, -1, dtype=np.int64)
        for v, want in enumerate(_order_variants(st, int(k) % 4)):
            if want is not None:
                bits = np.where((bits < 0) & (got == np.uint64(want)), v, bits)
        ob[sel] = bits
    if np.any(ob < 0):
        return None
    outer, swap = ob >> 1, ob & 1
    code = ((anchor + 1) | (s0.astype(np.int64) << 2) | (s1.astype(np.int64) << 4) | (outer << 6) | (swap << 7)
            | ((vec == 8).astype(np.int64) << 8) | ((flags & 1) << 9) | (((flags >> 1) & 1) << 10))
    return code.astype(np.uint16)


def _host_ctx():
    """Context for host-side library calls (enumeration/legality): the device
    context when a GPU is present, else a host-only context."""
    return _lib.host_context()


def candidate_actions(s):
    """All legal decisions for the next stage, in the reference's order
    (schedule_space.py:379-452), enumerated by the native library."""
    if s.is_complete:
        raise IllegalActionError("state is already complete")
    inf = _info(s.pipeline)
    ctx = _host_ctx()
    pid = ctx.pipeline_id(inf.desc)
    prefix = np.frombuffer(inf.records_of(s), dtype=_lib.DECISION_DTYPE)
    cap = 4096
    buf = np.zeros(cap, dtype=_lib.DECISION_DTYPE)
    n = ctypes.c_int64()
    ctx.check(ctx.lib.ts_candidates(ctx.h, pid, _lib._p(prefix) if len(prefix) else None,
                                    len(prefix), _lib._p(buf), cap, ctypes.byref(n)))
    idx = len(s.decisions)
    out = []
    if len(inf.enc_cache) >= (1 << 20):
        inf.enc_cache.clear()
    raw = buf[: n.value].tobytes()
    for i in range(n.value):
        rb = raw[16 * i:16 * i + 16]
        d = inf.decode_bytes(idx, rb)
        inf.enc_cache[id(d)] = (d, rb, idx)
        out.append(d)
    return out


def check_action(s, a) -> str | None:
    """None if legal, else the violated invariant (schedule_space.py:288-347)."""
    if s.is_complete:
        return "state is already complete"
    if a.stage != s.next_stage_name:
        return f"expected a decision for stage {s.next_stage_name!r}, got {a.stage!r}"
    inf = _info(s.pipeline)
    try:
        rec = np.frombuffer(inf.encode(len(s.decisions), a), dtype=_lib.DECISION_DTYPE)
    except IllegalActionError as e:
        return str(e)
    ctx = _host_ctx()
    pid = ctx.pipeline_id(inf.desc)
    prefix = np.frombuffer(inf.records_of(s), dtype=_lib.DECISION_DTYPE)
    rc = ctx.lib.ts_check_action(ctx.h, pid, _lib._p(prefix) if len(prefix) else None,
                                 len(prefix), _lib._p(rec))
    if rc == _lib.TS_OK:
        return None
    if rc == _lib.TS_ERR_ILLEGAL:
        return ctx.lib.ts_last_error(ctx.h).decode()
    ctx.check(rc)
    return None


def apply(s, a):
    """Extend a state by one decision (schedule_space.py:350-358)."""
    reason = check_action(s, a)
    if reason is not None:
        raise IllegalActionError(reason)
    inf = _info(s.pipeline)
    child = ScheduleState(s.pipeline, tuple(s.decisions) + (a,))
    child._cache["ts_records"] = inf.records_of(s) + inf.encode(len(s.decisions), a)
    return child


def child_state(s, a):
    """`apply` without the legality round trip, for actions that came out of
    candidate_actions(s)."""
    inf = _info(s.pipeline)
    child = ScheduleState(s.pipeline, tuple(s.decisions) + (a,))
    child._cache["ts_records"] = inf.records_of(s) + inf.encode(len(s.decisions), a)
    return child


def state_from_decisions(p, decisions):
    s = initial_state(p)
    for d in decisions:
        s = apply(s, d)
    return s


def read_schedule(p, text: str):
    decisions = [parse_layer_schedule(line) for line in text.splitlines()
                 if line.strip() and not line.lstrip().startswith("#")]
    return state_from_decisions(p, decisions)


def state_from_key(p, key: str):
    prefix = p.name + "/"
    if not key.startswith(prefix):
        raise PipelineError(f"key {key!r} does not belong to pipeline {p.name!r}")
    body = key[len(prefix):]
    return state_from_decisions(p, [parse_layer_schedule(t) for t in body.split(";") if t])


def default_action(s) -> LayerSchedule:
    st = s.pipeline.stage(s.next_stage_name)
    return LayerSchedule(st.name, (), tuple(d for d, _ in st.all_dims))
