"""CPU oracle for the V(s) scoring path - TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module, and only as the checker.  The product package never
imports it.

A restatement of the reference's algorithm, cited line by line (paths under
/root/reference/pkg/src/tensched):

* nests / invocations / per-invocation extents: schedule_space.py:176-285
* candidate enumeration order: schedule_space.py:361-452
* features: featurizer.py:44-107 (math.log2 = glibc log2, Python ints,
  Fraction for the recompute factor, cost_oracle.py:108-121, :162-169)
* normalization: featurizer.py:136-137
* LSTM forward: _recurrent_cy.pyx:20-66 via oracle/lstm_ref.c (same
  operation order, libm exp/tanh); V = math.exp(raw + target_scale),
  value_model.py:126/:154
* greedy: search.py:90-112, SearchRng: search.py:30-58
* checkpoint: value_model.py:296-376

Pinned against the reference itself: tests/golden/* were produced by
tools/make_golden.py, which runs the unmodified reference (oracle/_ref).
"""

from __future__ import annotations

import ctypes
import json
import math
import pathlib
import struct
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


# ------------------------------------------------------------------ actions
@dataclass(frozen=True)
class Act:
    """A LayerSchedule (schedule_space.py:37-56) with the same fields."""

    stage: str
    splits: tuple
    order: tuple
    vectorize_width: int = 1
    parallel: bool = False
    compute_at: tuple | None = None
    store_at: tuple | None = None

    def render(self):
        sp = ",".join(f"{d}:{f}" for d, f in self.splits) or "-"
        at = "root" if self.compute_at is None else "%s@%d" % self.compute_at
        st = "root" if self.store_at is None else "%s@%d" % self.store_at
        return (f"{self.stage} split={sp} order={','.join(self.order)} "
                f"vec={self.vectorize_width} par={int(self.parallel)} at={at} store={st}")


def as_act(d) -> Act:
    return Act(d.stage, tuple(d.splits), tuple(d.order), d.vectorize_width, bool(d.parallel),
               d.compute_at, d.store_at)


# ------------------------------------------------------------------ pipeline
class Pipe:
    """Static facts of a pipeline (duck-typed on the reference's Pipeline)."""

    def __init__(self, p):
        self.p = p
        self.by = {s.name: s for s in p.stages}
        names = [s.name for s in p.stages]
        deps = {s.name: [e.producer for e in s.inputs if e.producer in self.by] for s in p.stages}
        topo = []
        while len(topo) < len(names):  # pipeline_ir.py:179-204
            moved = False
            for n in names:
                if n not in topo and all(d in topo for d in deps[n]):
                    topo.append(n)
                    moved = True
            assert moved, "cycle"
        self.topo = topo
        self.sched = topo[::-1]  # pipeline_ir.py:207-213
        self.cons = {n: [s.name for s in p.stages if any(e.producer == n for e in s.inputs)]
                     for n in names}

    def elem(self, name):
        if name in self.by:
            return 4
        return next(b.element_size for b in self.p.buffers if b.name == name)


def _fp_extent(am, lo_hi):
    if am.consumer_dim is None:
        return am.window
    lo, hi = lo_hi[am.consumer_dim]
    return (am.stride * (hi - 1) + am.window) - am.stride * lo


def _loops(stage, pe, a: Act):
    """[(name, dim, extent)] in a.order (schedule_space.py:228-255)."""
    sp = dict(a.splits)
    named = {}
    for (d, _), e in zip(stage.dims, pe):
        if d in sp:
            named[d + "o"] = (d, e // sp[d])
            named[d + "i"] = (d, sp[d])
        else:
            named[d] = (d, e)
    for d, e in stage.reduction_dims:
        named[d] = (d, e)
    assert sorted(named) == sorted(a.order), (stage.name, a.order)
    return [(n,) + named[n] for n in a.order]


def _anchor_ok(loops, lvl):
    pos = {n: i for i, (n, _, _) in enumerate(loops)}
    for n, d, _ in loops:
        if n == d + "i" and d + "o" in pos and pos[n] <= lvl < pos[d + "o"]:
            return False
    return True


def _anchored(P: Pipe, nests, name, anchor):
    """(pe, inv, depth) under `anchor` (schedule_space.py:190-225)."""
    st = P.by[name]
    if anchor is None:
        return tuple(e for _, e in st.dims), 1, 0
    cname, lvl = anchor
    cloops, cinv, cdepth = nests[cname][3], nests[cname][1], nests[cname][2]
    inv = cinv
    for _, _, e in cloops[: lvl + 1]:
        inv *= e
    cst = P.by[cname]
    rem = {d: 1 for d, _ in cst.dims + cst.reduction_dims}
    for _, d, e in cloops[lvl + 1:]:
        rem[d] *= e
    region = [(0, rem[d]) for d, _ in cst.dims + cst.reduction_dims]
    pe = None
    for e in cst.inputs:
        if e.producer != name:
            continue
        ext = tuple(_fp_extent(am, region) for am in e.access)
        pe = ext if pe is None else tuple(max(x, y) for x, y in zip(pe, ext))
    return pe, inv, cdepth + lvl + 1


def nests_of(P: Pipe, decisions):
    """name -> (pe, inv, depth, loops) for every decision."""
    nests = {}
    for a in decisions:
        pe, inv, depth = _anchored(P, nests, a.stage, a.compute_at)
        nests[a.stage] = (pe, inv, depth, _loops(P.by[a.stage], pe, a))
    return nests


def candidates(P: Pipe, decisions):
    """candidate_actions (schedule_space.py:379-452), same order."""
    nests = nests_of(P, decisions)
    name = P.sched[len(decisions)]
    st = P.by[name]
    anchors = [None]
    if len(P.cons[name]) == 1 and P.cons[name][0] in nests:
        c = P.cons[name][0]
        cl = nests[c][3]
        anchors += [(c, l) for l in range(min(3, len(cl))) if _anchor_ok(cl, l)]
    sdims = [d for d, _ in st.dims[-2:]]
    rnames = [d for d, _ in st.reduction_dims]
    out = []
    for anchor in anchors:
        pe = dict(zip((d for d, _ in st.dims), _anchored(P, nests, name, anchor)[0]))
        choices = [[None] + [f for f in (8, 32) if pe[d] % f == 0 and f < pe[d]] for d in sdims]
        stores = [None] if anchor is None else [None, anchor]
        combos = [[]]
        for ch in choices:
            combos = [c + [x] for c in combos for x in ch]
        for combo in combos:
            splits = tuple((d, f) for d, f in zip(sdims, combo) if f is not None)
            sp = dict(splits)
            pnames, ext = [], {}
            for d, _ in st.dims:
                if d in sp:
                    pnames += [d + "o", d + "i"]
                    ext[d + "o"], ext[d + "i"] = pe[d] // sp[d], sp[d]
                else:
                    pnames.append(d)
                    ext[d] = pe[d]
            for d, e in st.reduction_dims:
                ext[d] = e
            orders = []
            for base in ([pnames + rnames, rnames + pnames] if rnames else [pnames]):
                for swap in (False, True):
                    seq = list(base)
                    if swap and len(seq) >= 2:
                        seq[-1], seq[-2] = seq[-2], seq[-1]
                    if tuple(seq) not in orders:
                        orders.append(tuple(seq))
            for order in orders:
                vecs = [1] + ([8] if order[-1] not in rnames and ext[order[-1]] % 8 == 0 else [])
                pars = [False] + ([True] if order[0] not in rnames else [])
                for v in vecs:
                    for par in pars:
                        for store in stores:
                            out.append(Act(name, splits, order, v, par, anchor, store))
    return out


# ------------------------------------------------------------------ features
def intrinsic_rows(P: Pipe) -> np.ndarray:
    """featurizer.py:44-65 via pipeline_ir.py:241-252."""
    rows = []
    for n in P.topo:
        st = P.by[n]
        full = [(0, e) for _, e in st.dims + st.reduction_dims]
        points = math.prod(e for _, e in st.dims) * math.prod(e for _, e in st.reduction_dims)
        flops = points * st.flops_per_point
        inb = sum(math.prod(_fp_extent(am, full) for am in e.access) * P.elem(e.producer)
                  for e in st.inputs)
        outb = math.prod(e for _, e in st.dims) * 4
        ov = 0.0
        for e in st.inputs:
            for am in e.access:
                ov = max(ov, am.window / max(1, am.stride))
        rows.append([math.log2(1 + points), math.log2(1 + flops), math.log2(1 + inb),
                     math.log2(1 + outb), flops / (1 + inb + outb), float(len(st.inputs)),
                     float(len(st.reduction_dims)), ov])
    return np.array(rows, dtype=np.float64)


def features(P: Pipe, decisions, cache_size=32768) -> np.ndarray:
    """[T,16] raw matrix (featurizer.py:68-107)."""
    mat = np.zeros((len(P.topo), 16))
    mat[:, :8] = intrinsic_rows(P)
    nests = nests_of(P, decisions)
    dec = {a.stage: a for a in decisions}
    for i, n in enumerate(P.topo):
        if n not in nests:
            continue
        pe, inv, depth, loops = nests[n]
        st, a = P.by[n], dec[n]
        red = math.prod(e for _, e in st.reduction_dims)
        dom = math.prod(e for _, e in st.dims) * red
        ppi = math.prod(pe) * red
        ws = 4 * (math.prod(e for _, e in st.dims) if a.store_at is None else math.prod(pe))
        par = loops[0][2] if a.parallel else 0
        mat[i, 8:] = [1.0, math.log2(a.vectorize_width), math.log2(par) if par else 0.0,
                      math.log2(loops[-1][2]), float(depth),
                      math.log2(float(Fraction(inv * ppi, dom))),
                      1.0 if ws <= cache_size else 0.0, math.log2(1 + inv)]
    return mat


def normalize(params, mat):
    return (mat - params["mean"]) / params["std"]


# ------------------------------------------------------------------ LSTM / V
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        so = HERE / "liboracle.so"
        if not so.exists():
            import subprocess
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        _LIB = ctypes.CDLL(str(so))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        _LIB.oracle_lstm_forward.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp, i64,
                                             ctypes.c_double, vp]
        _LIB.oracle_lstm_forward.restype = None
    return _LIB


def lstm_forward(X, Wx, Wh, b, w, b_out) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float64)
    B, T, F = X.shape
    H = len(w)
    out = np.empty(B)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (Wx, Wh, b, w)]
    p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    _lib().oracle_lstm_forward(p(X), B, T, F, *(p(a) for a in arrs), H, float(b_out), p(out))
    return out


def values(params, P: Pipe, states) -> np.ndarray:
    """V for a list of decision lists of one pipeline (value_model.py:129-155)."""
    if not states:
        return np.empty(0)
    X = np.stack([normalize(params, features(P, s)) for s in states])
    raw = lstm_forward(X, params["Wx"], params["Wh"], params["b"], params["w"], params["b_out"])
    return np.array([math.exp(r + params["target_scale"]) for r in raw])


def load_checkpoint(path) -> dict:
    """TSVM v1 (value_model.py:296-376)."""
    data = pathlib.Path(path).read_bytes()
    assert data[:4] == b"TSVM"
    version, hlen = struct.unpack("<II", data[4:12])
    assert version == 1
    hdr = json.loads(data[12:12 + hlen])
    H = hdr["hidden"]
    off = 12 + hlen
    out = {"hidden": H, "b_out": float.fromhex(hdr["b_out"]),
           "target_scale": float.fromhex(hdr["target_scale"])}
    for key, shape in (("Wx", (16, 4 * H)), ("Wh", (H, 4 * H)), ("b", (4 * H,)), ("w", (H,)),
                       ("mean", (16,)), ("std", (16,))):
        cnt = math.prod(shape)
        out[key] = np.frombuffer(data[off:off + 8 * cnt], dtype="<f8").reshape(shape).copy()
        off += 8 * cnt
    return out


# ------------------------------------------------------------------ search
class SplitMix:
    """SearchRng (search.py:30-58)."""

    def __init__(self, seed):
        self.state = seed & MASK64

    def next_u64(self):
        self.state = (self.state + GAMMA) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, lo, hi):
        return lo + ((self.next_u64() >> 11) / float(1 << 53)) * (hi - lo)

    def randrange(self, n):
        return (self.next_u64() * n) >> 64


def greedy(P: Pipe, params, epsilon=0.0, rng=None):
    """search.py:90-112 with the oracle V; returns (decisions, visited)."""
    decisions, visited = [], 0
    while len(decisions) < len(P.topo):
        cands = candidates(P, decisions)
        visited += len(cands)
        vals = list(values(params, P, [decisions + [a] for a in cands]))
        if epsilon > 0:
            vals = [v * (1.0 + rng.uniform(-epsilon, epsilon)) for v in vals]
        best = min(range(len(vals)), key=lambda i: (vals[i], i))
        decisions.append(cands[best])
    return decisions, visited


def beam(P: Pipe, params, prefix, width):
    """search.py:115-133 with the oracle V: children of every frontier state
    in frontier order, ranked by (v, index), the `width` best kept; the
    final V(frontier) argmin by (v, index).  Returns the decisions."""
    frontier = [list(prefix)]
    while len(frontier[0]) < len(P.topo):
        children = [f + [a] for f in frontier for a in candidates(P, f)]
        vals = list(values(params, P, children))
        ranked = sorted(range(len(children)), key=lambda i: (float(vals[i]), i))
        frontier = [children[i] for i in ranked[:width]]
    vals = list(values(params, P, frontier))
    return frontier[min(range(len(frontier)), key=lambda i: (float(vals[i]), i))]


def random_partial(P: Pipe, seed: int):
    """Synthetic-sweep state: SearchRng(seed), d = randrange(T) + 1, then d
    uniform candidate choices (search.py:136-142 variant)."""
    rng = SplitMix(seed)
    d = rng.randrange(len(P.topo)) + 1
    decisions = []
    for _ in range(d):
        c = candidates(P, decisions)
        decisions.append(c[rng.randrange(len(c))])
    return decisions


# ------------------------------------------------------------------ training
def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def gradients(params, X_list, logt, n_total=None):
    """value_model.gradients (value_model.py:182-210) for a list of
    normalized matrices grouped by length (ascending), via the numpy BPTT of
    _recurrent_np.py:38-96.  Returns the flat [Wx|Wh|b|w|b_out] gradient."""
    Wx, Wh, b, w, b_out = params["Wx"], params["Wh"], params["b"], params["w"], params["b_out"]
    H = len(w)
    n = len(X_list) if n_total is None else n_total
    gWx, gWh, gb, gw, gbo = np.zeros_like(Wx), np.zeros_like(Wh), np.zeros(4 * H), np.zeros(H), 0.0
    groups = {}
    for m, lt in zip(X_list, logt):
        groups.setdefault(m.shape[0], []).append((m, lt))
    for T, items in sorted(groups.items()):
        X = np.stack([m for m, _ in items])
        lt = np.array([v for _, v in items])
        B = X.shape[0]
        h, c = np.zeros((B, H)), np.zeros((B, H))
        raw = np.full(B, T * b_out)
        cache = []
        for t in range(T):
            z = X[:, t, :] @ Wx + h @ Wh + b
            i, f = _sigmoid(z[:, :H]), _sigmoid(z[:, H:2 * H])
            g, o = np.tanh(z[:, 2 * H:3 * H]), _sigmoid(z[:, 3 * H:])
            c_prev, h_prev = c, h
            c = f * c + i * g
            tc = np.tanh(c)
            h = o * tc
            raw += h @ w
            cache.append((i, f, g, o, c_prev, h_prev, tc, h))
        d_raw = 2.0 * (raw + params["target_scale"] - lt) / n
        gbo += T * d_raw.sum()
        dh_next, dc_next = np.zeros((B, H)), np.zeros((B, H))
        for t in range(T - 1, -1, -1):
            i, f, g, o, c_prev, h_prev, tc, h = cache[t]
            gw += h.T @ d_raw
            dh = w[None, :] * d_raw[:, None] + dh_next
            do = dh * tc
            dc = dc_next + dh * o * (1.0 - tc * tc)
            di, df, dg = dc * g, dc * c_prev, dc * i
            dc_next = dc * f
            dz = np.concatenate([di * i * (1 - i), df * f * (1 - f), dg * (1 - g * g),
                                 do * o * (1 - o)], axis=1)
            gWx += X[:, t, :].T @ dz
            gWh += h_prev.T @ dz
            gb += dz.sum(axis=0)
            dh_next = dz @ Wh.T
    return np.concatenate([gWx.ravel(), gWh.ravel(), gb, gw, [gbo]])
