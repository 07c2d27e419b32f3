"""Host-side logic of the product (no GPU): the C-ABI library loads and
exports every declared symbol, the host mirror parses/encodes like the
reference, native candidate enumeration and legality match the golden
vectors, and the shared nest/feature core (csrc/ts_core.cuh, host build)
reproduces the reference's feature matrices bit for bit."""

import ctypes
import math
import pathlib
import random
import re

import numpy as np
import pytest

from helpers import bits, pipeline_from, product_states
from paper_2011_14486_b200 import _lib
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.errors import IllegalActionError, ParseError

ROOT = pathlib.Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    header = (ROOT / "include" / "tensched_b200.h").read_text()
    names = re.findall(r"^\s*(?:int|void|const char\*|int64_t|void\*)\s+\**(ts_\w+)\(", header, re.M)
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ts_abi_version() == 1


def test_pointer_keeps_temporary_alive():
    """_lib._p(temporary) must keep the array alive until the C call: a bare
    address let numpy free `T.copy()` before ts_train_load read it (a
    training run on corrupted depths, seen as a rare flaky parity failure)."""
    import gc
    p = _lib._p(np.arange(1000, dtype=np.int32).copy())
    gc.collect()
    junk = [np.full(1000, -7, dtype=np.int32) for _ in range(64)]  # reuse freed blocks
    view = ctypes.cast(p, ctypes.POINTER(ctypes.c_int32))
    assert [view[i] for i in (0, 1, 500, 999)] == [0, 1, 500, 999]
    del junk


def test_host_only_context_refuses_device_work():
    ctx = _lib.Context(-1)
    out = np.zeros(1)
    rc = ctx.lib.ts_score_states(ctx.h, 0, None, _lib._p(np.zeros(2, np.int64)), 1, 0, _lib._p(out))
    assert rc != 0


def test_parse_and_topo_match_reference(greedy_golden):
    import oracle as O
    for key, g in greedy_golden.items():
        p = pipeline_from(g)
        assert p.name == g["pipeline"]
        assert pi.topological_order(p) == O.Pipe(p).topo


def test_parse_errors():
    with pytest.raises(ParseError):
        pi.parse_pipeline("pipeline x\nstage a dims x:4 flops 1\n  in z map x*1+1\n")
    with pytest.raises(ParseError):
        pi.parse_pipeline("stage a dims x:4 flops 1\n")


def test_candidates_match_golden(candidates_golden, greedy_golden):
    for key, walk in candidates_golden.items():
        p = pipeline_from(greedy_golden[key])
        rng = random.Random(0)
        s = ss.initial_state(p)
        r5 = __import__("oracle").SplitMix(5)
        for step in walk:
            c = ss.candidate_actions(s)
            assert [a.render() for a in c] == step, (key, len(s.decisions))
            s = ss.apply(s, c[r5.randrange(len(c))])


def _fresh(d, **kw):
    """A new decision object equal to d (or with fields replaced)."""
    import dataclasses
    return dataclasses.replace(d, **kw)


def test_native_encoder_matches_python(candidates_golden, greedy_golden):
    """csrc/hostenc.c's encode_native against _PipelineInfo._encode_fields on
    every candidate of the golden walks (fresh objects, empty caches: no
    call may reach the Python encoder), and every illegal mutation going to
    the Python encoder and raising its error."""
    from paper_2011_14486_b200 import _hostenc
    n_legal = n_bad = 0
    for key, walk in candidates_golden.items():
        p = pipeline_from(greedy_golden[key])
        inf = ss._info(p)
        s = ss.initial_state(p)
        r5 = __import__("oracle").SplitMix(5)
        for _ in walk:
            j = len(s.decisions)
            cands = ss.candidate_actions(s)
            calls = []

            def fallback(idx, d):
                calls.append(idx)
                return inf.encode(idx, d)

            children = [ss.ScheduleState(p, (*s.decisions, _fresh(a))) for a in cands]
            _hostenc.clear()
            rb, _ = _hostenc.encode_group(children, list(range(len(children))), inf.T, fallback, {}, inf.stab)
            want = b"".join(b"".join(inf._encode_fields(i, d) for i, d in enumerate(c.decisions))
                            for c in children)
            assert rb == want, key
            if inf.stab[j] is not None:
                assert not calls, (key, j)
            n_legal += len(children)
            a = cands[0]
            st = inf.stages[j]
            bad = [_fresh(a, stage=a.stage + "_x"), _fresh(a, vectorize_width=0),
                   _fresh(a, vectorize_width=256), _fresh(a, order=a.order[:-1]),
                   _fresh(a, order=(*a.order[:-1], a.order[0])), _fresh(a, splits=((st.dims[0][0], 1),)),
                   _fresh(a, splits=((st.dims[0][0], 256),)), _fresh(a, splits=(("nope", 2),)),
                   _fresh(a, compute_at=("nope", 0)), _fresh(a, store_at=("nope", 1))]
            if a.compute_at is not None:
                bad += [_fresh(a, compute_at=(a.compute_at[0], 8)),
                        _fresh(a, store_at=(a.compute_at[0], a.compute_at[1] + 1))]
            for d in bad:
                child = ss.ScheduleState(p, (*s.decisions, d))
                try:
                    inf._encode_fields(j, d)
                    want_err = None
                except Exception as e:  # the reference's error for this decision
                    want_err = (type(e), str(e))
                _hostenc.clear()
                if want_err is None:  # a mutation that is still legal
                    rb, _ = _hostenc.encode_group([child], [0], inf.T, inf.encode, {}, inf.stab)
                    assert rb[-16:] == inf._encode_fields(j, d)
                    continue
                with pytest.raises(want_err[0]) as ei:
                    _hostenc.encode_group([child], [0], inf.T, inf.encode, {}, inf.stab)
                assert str(ei.value) == want_err[1]
                n_bad += 1
            s = ss.apply(s, cands[r5.randrange(len(cands))])
    assert n_legal > 1000 and n_bad > 100, (n_legal, n_bad)


def test_encode_decode_roundtrip(state_sets):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        states = product_states(p, z["keys"][:6])
        for inf, idxs, recs, offs in ss.encode_states(states):
            for j, i in enumerate(idxs):
                dec = [inf.decode(k, r) for k, r in enumerate(recs[offs[j]:offs[j + 1]])]
                assert [d.render() for d in dec] == [d.render() for d in states[i].decisions]


def test_action_codes_roundtrip_every_candidate(candidates_golden, greedy_golden):
    """Every decision candidate_actions produces along the golden walks has a
    16-bit action code, and the native decoder (the featurizer's) turns the
    codes back into the identical 16-byte records."""
    ctx = _lib.host_context()
    for key, walk in candidates_golden.items():
        p = pipeline_from(greedy_golden[key])
        s = ss.initial_state(p)
        r5 = __import__("oracle").SplitMix(5)
        children = []
        for _ in walk:
            c = ss.candidate_actions(s)
            children += [ss.apply(s, a) for a in c]
            s = ss.apply(s, c[r5.randrange(len(c))])
        for inf, idxs, recs, offs in ss.encode_states(children):
            codes = ss.action_codes(inf, recs, offs)
            assert codes is not None, key
            depths = np.diff(offs).astype(np.uint8)
            out = np.zeros(len(recs), dtype=_lib.DECISION_DTYPE)
            pid = ctx.pipeline_id(inf.desc)
            ctx.check(ctx.lib.ts_decode_codes(ctx.h, pid, _lib._p(codes), _lib._p(depths), len(idxs),
                                              _lib._p(out)))
            assert out.tobytes() == recs.tobytes(), key
            back = np.zeros(len(recs), dtype=np.uint16)  # native encoder == python encoder
            ctx.check(ctx.lib.ts_encode_codes(ctx.h, pid, _lib._p(recs), _lib._p(depths), len(idxs),
                                              _lib._p(back)))
            assert np.array_equal(back, codes), key


def test_action_codes_reject_decisions_outside_the_space(greedy_golden):
    p = pipeline_from(greedy_golden["ref:pipelines/toys/t2_stencil.pl"])
    s0 = ss.initial_state(p)
    name = ss._info(p).sched[0]
    for odd in (ss.LayerSchedule(name, (("x", 4),), ("xo", "xi")),   # factor outside SPLIT_FACTORS
                ss.LayerSchedule(name, (), ("x",), 4)):               # width outside VEC_WIDTHS
        assert ss.check_action(s0, odd) is None
        [(inf, idxs, recs, offs)] = ss.encode_states([ss.apply(s0, odd)])
        assert ss.action_codes(inf, recs, offs) is None


def test_check_action_rejects_illegal(greedy_golden):
    p = pipeline_from(greedy_golden["ref:pipelines/toys/t2_stencil.pl"])
    s = ss.initial_state(p)
    blur = ss.LayerSchedule("blur", (("x", 8),), ("xo", "xi"), 1, False, None, None)
    s = ss.apply(s, blur)
    bad = [
        ss.LayerSchedule("pre", (("x", 7),), ("xo", "xi")),             # does not divide 66
        ss.LayerSchedule("pre", (), ("x",), 3),                          # bad width
        ss.LayerSchedule("pre", (), ("x",), 1, False, ("blur", 5)),      # no such level
        ss.LayerSchedule("pre", (), ("x",), 1, False, None, ("blur", 0)),  # store without compute
        ss.LayerSchedule("blur", (), ("x",)),                            # wrong stage
    ]
    for a in bad:
        assert ss.check_action(s, a) is not None, a
        with pytest.raises(IllegalActionError):
            ss.apply(s, a)
    ok = ss.LayerSchedule("pre", (), ("x",), 1, False, ("blur", 0), ("blur", 0))
    assert ss.check_action(s, ok) is None


def test_descriptor_envelope(greedy_golden):
    for g in greedy_golden.values():
        d = pi.descriptor(pipeline_from(g))
        assert d[0] == pi.DESC_MAGIC and d.size == 4 + d[1] * pi.DESC_STAGE_WORDS
        assert 0 <= d[2] <= 16


def test_native_core_log2_matches_libm(native_core):
    for i in range(1, 1 << 17):
        assert native_core.core_log2(float(i)) == math.log2(i)
    rng = random.Random(7)
    for _ in range(20000):
        x = rng.random() * 2.0 ** rng.randint(-40, 80)
        if x > 0:
            assert native_core.core_log2(x) == math.log2(x)


def test_native_core_bigint_rounding(native_core):
    rng = random.Random(3)

    def limbs(n):
        return np.array([(n >> (64 * k)) & ((1 << 64) - 1) for k in range(4)], dtype=np.uint64)

    for _ in range(20000):
        n = rng.getrandbits(rng.randint(1, 200)) + 1
        d = rng.getrandbits(rng.randint(1, 63)) + 1
        a = limbs(n)
        assert native_core.core_div(a.ctypes.data, d) == n / d
        assert native_core.core_to_double(a.ctypes.data) == float(n)
        tie = ((rng.getrandbits(52) | (1 << 52)) * 2 + 1) << rng.randint(0, 150)
        assert native_core.core_to_double(limbs(tie).ctypes.data) == float(tie)


def test_native_core_div128_correctly_rounded(native_core):
    """The 128-bit division path of the recompute feature equals CPython's
    int/int true division, including exact halfway cases."""
    rng = random.Random(11)
    M = (1 << 64) - 1
    for _ in range(100000):
        n = rng.getrandbits(rng.randint(1, 127)) + 1
        d = rng.getrandbits(rng.randint(1, 63)) + 1
        assert native_core.core_div128(n & M, n >> 64, d) == n / d, (n, d)
    for _ in range(20000):  # ties: n/d = (odd 54-bit) / 2 * 2^e
        d = rng.getrandbits(rng.randint(1, 40)) + 1
        q = ((rng.getrandbits(52) | (1 << 52)) * 2 + 1)
        n = q * d << rng.randint(0, 10)
        if n < (1 << 127):
            assert native_core.core_div128(n & M, n >> 64, d * 2) == n / (d * 2)


def test_native_core_log2_1p_invocations(native_core):
    """f15 = log2(1 + inv) (PyLong_AsDouble then libm log2) for invocation
    counts across 64-, 128- and 256-bit paths."""
    rng = random.Random(5)
    M = (1 << 64) - 1
    for _ in range(20000):
        inv = rng.getrandbits(rng.randint(1, 127))
        assert native_core.core_log2_1p(inv & M, inv >> 64) == math.log2(1 + inv), inv
    for hi_bits in range(1, 65):  # exact boundaries of the top-64 extraction
        inv = (1 << (63 + hi_bits)) - 1
        assert native_core.core_log2_1p(inv & M, inv >> 64) == math.log2(1 + inv)


def test_native_core_features_bit_exact(state_sets, native_core):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        states = product_states(p, z["keys"])
        for inf, idxs, recs, offs in ss.encode_states(states):
            out = np.empty((len(idxs), inf.T, 16))
            rc = native_core.core_featurize(inf.desc.ctypes.data, inf.desc.size,
                                            recs.ctypes.data, offs.ctypes.data, len(idxs),
                                            out.ctypes.data)
            assert rc == 0
            assert np.array_equal(bits(out), bits(z["features"][idxs])), name


def test_glibc_log2_exact_on_powers_of_two(native_core):
    """The device log2 short-circuits powers of two to their exponent; glibc
    returns them exactly (all normal and subnormal powers)."""
    for k in range(-1074, 1024):
        x = 2.0 ** k
        assert math.log2(x) == k
        assert native_core.core_log2(x) == k


def test_glibc_exp_tanh_ports_bit_exact(native_core):
    """The exact leg's exp / tanh (csrc/ts_glibc_math.cuh: glibc 2.39's
    __exp_fma and fdlibm tanh over __expm1_fma, restated) against this host's
    libm through CPython's math.exp / math.tanh - the functions behind the
    reference's Cython kernel and predict_states (_recurrent_cy.pyx:17-18,
    :58-60, value_model.py:154) - bit for bit on 400k values over the LSTM's
    ranges, both tanh forms, exp's special cases and the subnormal range."""
    import ctypes
    import math
    rng = np.random.default_rng(3)
    xs = np.concatenate([
        rng.uniform(-30, 30, 150_000), rng.uniform(-2, 2, 100_000), rng.uniform(-760, 760, 50_000),
        rng.uniform(-1, 1, 50_000) * np.exp2(-rng.integers(0, 60, 50_000)),
        np.exp2(rng.integers(-5, 10, 10_000)) * (1 + rng.uniform(-1e-9, 1e-9, 10_000)),
        [0.0, -0.0, 1.0, -1.0, 22.0, -22.0, 512.0, -512.0, 709.78, -745.1, -708.5, 1e-300, 5e-324,
         0.34657359027997264, 1.0397207708399179, 38.816242111356935, 44.0, -0.25, 0.5],
    ]).astype(np.float64)
    out = np.empty(2 * len(xs))
    native_core.core_exp_tanh(xs.ctypes.data_as(ctypes.c_void_p), len(xs), out.ctypes.data_as(ctypes.c_void_p))
    want_e = np.array([math.exp(x) if x < 709.7 else float("inf") for x in xs])
    want_t = np.array([math.tanh(x) for x in xs])
    fin = xs < 709.7  # math.exp raises OverflowError beyond; the port returns inf like libm
    assert np.array_equal(out[0::2][fin].view(np.uint64), want_e[fin].view(np.uint64))
    assert np.array_equal(out[1::2].view(np.uint64), want_t.view(np.uint64))


def test_glibc_tanh_branch_free_form(native_core):
    """glibc_tanh_bf (one expm1 per lane, selects instead of branches - what
    the exact LSTM kernels run) equals libm tanh bit for bit."""
    import ctypes
    import math
    rng = np.random.default_rng(4)
    xs = np.concatenate([rng.uniform(-30, 30, 200_000), rng.uniform(-2.5, 2.5, 200_000),
                         rng.uniform(-1, 1, 50_000) * np.exp2(-rng.integers(0, 60, 50_000)),
                         np.array([0.0, -0.0, 1.0, -1.0, 22.0, -22.0, 0.17328679513998632, 0.5198603854199589,
                                   0.9999999999999999, 19.4, 1e-17, -1e-17, 5e-324])])
    out = np.empty(len(xs))
    native_core.core_tanh_bf(xs.ctypes.data_as(ctypes.c_void_p), len(xs), out.ctypes.data_as(ctypes.c_void_p))
    want = np.array([math.tanh(x) for x in xs])
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


def test_native_host_encoder_matches_python_path(greedy_golden):
    """csrc/hostenc.c (identity-cached decision records, one C call per
    pipeline group) returns exactly the Python path's records and offsets, on
    states sharing decision objects (search children), on repeated state
    objects, and raises the same errors."""
    assert ss._hostenc is not None, "the native host encoder is not built"
    ss._hostenc.clear()
    g = greedy_golden["assets/pipelines/nets/vgg16.pl"]
    p = pi.parse_pipeline(g["text"])
    s = ss.initial_state(p)
    states = []
    for k, r in enumerate(g["schedule"]):
        cands = ss.candidate_actions(s)
        states.extend(ss.child_state(s, a) for a in cands[:5])  # children share the parent's objects
        s = ss.apply(s, ss.parse_layer_schedule(r))
    states += states[:7]  # repeated objects
    native = ss.encode_states(states)
    saved, ss._hostenc = ss._hostenc, None
    try:
        for st in states:
            st._cache.pop("ts_records", None)
        python = ss.encode_states(states)
    finally:
        ss._hostenc = saved
    assert len(native) == len(python) == 1
    assert np.array_equal(native[0][2].view(np.uint8), python[0][2].view(np.uint8))
    assert np.array_equal(native[0][3], python[0][3])
    bad = ss.ScheduleState(p, tuple(ss.initial_state(p).decisions) + (ss.LayerSchedule("nope", (), ("x",)),))
    with pytest.raises(IllegalActionError):
        ss.encode_states([bad])


def test_native_host_encoder_caches_are_per_pipeline(greedy_golden):
    """A record depends on the pipeline (the stage's loop table, its sole
    consumer), so the native encoder's identity and value caches must not
    carry a decision across pipelines: t3_chain's conv decision
    compute_at=(relu, 0) is legal there and illegal in a variant where pool
    also reads conv - reusing the same decision objects, or equal ones, must
    still raise in the variant (schedule_space.py:299-305 sole-consumer
    rule)."""
    import dataclasses

    assert ss._hostenc is not None, "the native host encoder is not built"
    text = greedy_golden["ref:pipelines/toys/t3_chain.pl"]["text"]
    a = pi.parse_pipeline(text)
    b = pi.parse_pipeline(text.replace("in relu map x*2+2", "in relu map x*2+2\n  in conv map x*2+1"))
    s = ss.initial_state(a)
    for _ in range(3):
        s = ss.apply(s, ss.candidate_actions(s)[-1])
    assert s.decisions[2].compute_at == ("relu", 0)
    copies = tuple(dataclasses.replace(d) for d in s.decisions)
    for decs in (s.decisions, copies):  # fresh states: no cached records, the tables fill
        recs = ss.encode_states([ss.ScheduleState(a, decs)])[0][2]
        assert list(recs["anchor"]) == [-1, 1, 0]
    for decs in (s.decisions, copies):
        with pytest.raises(IllegalActionError, match="sole consumer"):
            ss.encode_states([ss.ScheduleState(b, decs)])


def test_fast_leg_tanh_rational_accuracy():
    """The FAST leg's cell tanh (csrc/ts_lstm_tc.cuh, TS_RAT_TANH): the
    odd/even rational in fp32 with the kernel's clamp, Horner order and
    coefficients, against libm tanh - |error| < 5e-7 everywhere."""
    import re as _re
    src = (pathlib.Path(__file__).resolve().parent.parent / "paper_2011_14486_b200" / "csrc" /
           "ts_lstm_tc.cuh").read_text()
    k = {m.group(1): np.float32(float(m.group(2).rstrip("f")))
         for m in _re.finditer(r"\b(kT(?:A|B)\d+|kTanhClamp) = ([-0-9.e+]+f)", src)}
    f32 = np.float32
    x = np.linspace(-12.0, 12.0, 400001).astype(f32)
    xc = np.clip(x, -k["kTanhClamp"], k["kTanhClamp"]).astype(f32)
    x2 = (xc * xc).astype(f32)
    p = k["kTA13"]
    for c in ("kTA11", "kTA9", "kTA7", "kTA5", "kTA3", "kTA1"):
        p = (p * x2 + k[c]).astype(f32)
    p = (p * xc).astype(f32)
    q = k["kTB6"]
    for c in ("kTB4", "kTB2", "kTB0"):
        q = (q * x2 + k[c]).astype(f32)
    assert q.min() > 0.004 and q.max() < 0.95  # the shared reciprocal's range argument
    err = np.abs((p / q).astype(np.float64) - np.tanh(x.astype(np.float64)))
    assert err.max() < 5e-7, err.max()
