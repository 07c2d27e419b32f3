"""Parity of the sm_100a path against the reference's golden vectors and the
CPU oracle.  Every call goes through the C-ABI library (libtensched_b200.so).

Tolerances: features are bit-exact; V in EXACT mode (fp64, Cython op order,
glibc 2.39's exp/tanh restated) bit-exact as well; V in FAST mode
(tensor cores) within 1e-4 relative (BASELINE.json north_star, fp32 leg);
greedy schedules and visited counts identical."""

import numpy as np
import pytest

import oracle as O
from helpers import bits, oracle_decisions, oracle_params, pipeline_from, product_states
from paper_2011_14486_b200 import _lib
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.featurizer import featurize_states
from paper_2011_14486_b200.search import (NoiseConfig, SearchRng, greedy_schedule,
                                          greedy_schedule_gpu, model_value)
from paper_2011_14486_b200.value_model import MODE_EXACT, MODE_FAST, load, predict_states

pytestmark = pytest.mark.gpu

EXACT_RTOL = 1e-12
FAST_RTOL = 1e-4


@pytest.fixture(scope="module")
def v0(v0_path):
    return load(v0_path)


def test_features_bit_exact(state_sets, gpu_ctx):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        got = np.stack(featurize_states(product_states(p, z["keys"])))
        assert np.array_equal(bits(got), bits(z["features"])), name


def test_values_exact(state_sets, v0):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        got = predict_states(v0, product_states(p, z["keys"]), mode=MODE_EXACT)
        assert np.array_equal(bits(got), bits(z["values"])), name


def test_lstm_forward_exact(golden, v0):
    from paper_2011_14486_b200.backend import lstm_forward
    z = np.load(golden / "lstm_forward.npz")
    raw = lstm_forward(z["X"], v0.Wx, v0.Wh, v0.b, v0.w, v0.b_out)
    assert np.array_equal(bits(raw), bits(z["raw"]))


def test_position_and_batch_independence(state_sets, v0):
    z = state_sets["vgg16"]
    p = pipeline_from(z)
    states = product_states(p, z["keys"])
    one = np.array([predict_states(v0, [s])[0] for s in states[:6]])
    mixed = states[::-1] + states[:6]
    many = predict_states(v0, mixed)
    assert np.array_equal(bits(many[-6:]), bits(one))
    assert np.array_equal(bits(many[: len(states)][::-1][:6]), bits(one))


def test_greedy_fused_matches_reference(greedy_golden, v0):
    for key, g in greedy_golden.items():
        p = pipeline_from(g)
        s, visited, v = greedy_schedule_gpu(p, v0, return_value=True)
        assert [d.render() for d in s.decisions] == g["schedule"], key
        # the schedule file `cmd_schedule` writes (schedule_space.py:479-481), byte for byte
        assert ss.write_schedule(s) == "\n".join(g["schedule"]) + "\n", key
        assert visited == g["visited"], key
        assert v == float.fromhex(g["predicted"]), key


def test_greedy_generic_v_callable(greedy_golden, v0):
    for key in ("ref:pipelines/toys/t3_chain.pl", "ref:pipelines/deep/p12_deep.pl",
                "assets/pipelines/nets/crp2d.pl"):
        g = greedy_golden[key]
        s, visited = greedy_schedule(pipeline_from(g), model_value(v0))
        assert [d.render() for d in s.decisions] == g["schedule"], key
        assert visited == g["visited"]


def test_noisy_greedy(noisy_golden, greedy_golden, v0):
    for key, g in noisy_golden.items():
        base, seed = key.split("#")
        p = pipeline_from(greedy_golden[base])
        rng = SearchRng(int(seed))
        s, visited = greedy_schedule_gpu(p, v0, NoiseConfig(0.25), rng)
        assert [d.render() for d in s.decisions] == g["schedule"], key
        assert visited == g["visited"] and rng.state == g["rng_state"], key


def test_device_generator_matches_oracle_walk(state_sets, gpu_ctx):
    import ctypes
    import torch
    for name in ("t3_chain", "p12_deep", "vgg16", "resnet18"):
        z = state_sets[name]
        p = pipeline_from(z)
        inf = ss._info(p)
        pid = gpu_ctx.pipeline_id(inf.desc)
        n = len(z["seeds"])
        recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
        offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        nrec = ctypes.c_int64()
        gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(
            gpu_ctx.h, pid, int(z["seeds"][0]), n, recs.data_ptr(), offs.data_ptr(),
            ctypes.byref(nrec)))
        hr = np.frombuffer(recs[: nrec.value * 16].cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
        ho = offs.cpu().numpy()
        for i in range(n):
            dec = [inf.decode(k, r).render() for k, r in enumerate(hr[ho[i]:ho[i + 1]])]
            assert p.name + "/" + ";".join(dec) == str(z["keys"][i]), (name, i)


def test_fast_mode_within_tolerance(state_sets, v0):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        states = product_states(p, z["keys"])
        fast = predict_states(v0, states, mode=MODE_FAST)
        np.testing.assert_allclose(fast, z["values"], rtol=FAST_RTOL, atol=0, err_msg=name)


def test_oracle_agrees_on_fresh_states(v0_path, v0, greedy_golden):
    params = oracle_params(v0_path)
    p = pipeline_from(greedy_golden["assets/pipelines/nets/vgg16.pl"])
    P = O.Pipe(p)
    decs = [O.random_partial(P, seed) for seed in range(1000, 1024)]
    want = O.values(params, P, decs)
    states = [ss.state_from_decisions(p, d) for d in decs]
    assert np.array_equal(bits(predict_states(v0, states)), bits(want))
    feats = np.stack(featurize_states(states))
    for i, d in enumerate(decs):
        assert np.array_equal(bits(feats[i]), bits(O.features(P, d)))


def test_fast_mode_position_and_batch_independence(state_sets, v0):
    """Tiles replay the shared prefix: a state's FAST value must not depend on
    which tile (depth mix) it lands in."""
    z = state_sets["vgg16"]
    p = pipeline_from(z)
    states = product_states(p, z["keys"])
    alone = np.array([predict_states(v0, [s], mode=MODE_FAST)[0] for s in states[:8]])
    mixed = predict_states(v0, states[::-1] + states[:8] + states * 5, mode=MODE_FAST)
    assert np.array_equal(bits(mixed[len(states): len(states) + 8]), bits(alone))
    assert np.array_equal(bits(mixed[: len(states)][::-1][:8]), bits(alone))


def test_fast_mode_large_batch_matches_exact(gpu_ctx, v0):
    """1e5 device-generated VGG-16 states: FAST within 1e-4 of EXACT."""
    import ctypes
    import torch
    p = pipeline_from({"text": (__import__("pathlib").Path(__file__).resolve().parent.parent
                                / "assets/pipelines/nets/vgg16.pl").read_text()})
    inf = ss._info(p)
    pid = gpu_ctx.pipeline_id(inf.desc)
    gpu_ctx.set_params(v0)
    n = 100_000
    recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nrec = ctypes.c_int64()
    gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 777, n, recs.data_ptr(),
                                                        offs.data_ptr(), ctypes.byref(nrec)))
    out = {}
    for mode in (MODE_EXACT, MODE_FAST):
        o = torch.empty(n, dtype=torch.float64, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(),
                                                         offs.data_ptr(), n, nrec.value, mode,
                                                         o.data_ptr()))
        out[mode] = o.cpu().numpy()
    assert np.all(out[MODE_EXACT] > 0)
    np.testing.assert_allclose(out[MODE_FAST], out[MODE_EXACT], rtol=FAST_RTOL, atol=0)
    # batch-size independence across the LSTM kernel's variants (1, 2 or 4
    # tiles per CTA, chosen by the batch's tile count): prefixes of the batch
    # give bit-identical FAST values
    for m in (3_000, 30_000, 100_000):
        o = torch.empty(m, dtype=torch.float64, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), m,
                                                         int(offs[m].item()), MODE_FAST, o.data_ptr()))
        assert np.array_equal(bits(o.cpu().numpy()), bits(out[MODE_FAST][:m])), m


def test_reference_greedy_with_gpu_v_callable(greedy_golden, v0_path):
    """INTEGRATION.md level 1: the unmodified reference's greedy_schedule
    driven by the device V-callable, on the reference's own objects."""
    import pathlib
    import sys
    ref = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref"
    if not (ref / "tensched").exists():
        pytest.skip("oracle/_ref (the built reference) is not present")
    sys.path.insert(0, str(ref))
    from tensched.pipeline_ir import parse_pipeline as ref_parse
    from tensched.search import greedy_schedule as ref_greedy
    from tensched.value_model import load as ref_load
    from paper_2011_14486_b200.search import model_value as gpu_model_value
    params = ref_load(v0_path)
    for key in ("ref:pipelines/toys/t5_diamond.pl", "ref:pipelines/deep/p12_deep.pl"):
        g = greedy_golden[key]
        s, visited = ref_greedy(ref_parse(g["text"]), gpu_model_value(params))
        assert [d.render() for d in s.decisions] == g["schedule"] and visited == g["visited"]


def test_packed_wire_format_matches(state_sets, v0):
    """ts_score_states_packed (8-byte decisions + u8 depths) == ts_score_states."""
    from paper_2011_14486_b200 import _lib
    z = state_sets["vgg16"]
    p = pipeline_from(z)
    states = product_states(p, z["keys"]) * 100
    ctx = _lib.context(0)
    ctx.set_params(v0)
    for inf, idxs, recs, offsets in ss.encode_states(states):
        pid = ctx.pipeline_id(inf.desc)
        packed = _lib.pack_records(recs)
        depths = np.diff(offsets).astype(np.uint8)
        for mode in (MODE_EXACT, MODE_FAST):
            a = np.empty(len(idxs))
            b = np.empty(len(idxs))
            ctx.check(ctx.lib.ts_score_states(ctx.h, pid, _lib._p(recs), _lib._p(offsets), len(idxs),
                                              mode, _lib._p(a)))
            ctx.check(ctx.lib.ts_score_states_packed(ctx.h, pid, _lib._p(packed), _lib._p(depths),
                                                     len(idxs), mode, _lib._p(b)))
            assert np.array_equal(bits(a), bits(b))


@pytest.mark.gpu
def test_coded_wire_format_matches(gpu_ctx, v0):
    """ts_score_states_coded (16-bit action codes decoded in the featurizer +
    u8 depths) == ts_score_states on 2e5 device-generated VGG-16 states, both
    modes, bit for bit; several chunkings; an out-of-space code is reported."""
    import ctypes
    import os
    import torch
    from paper_2011_14486_b200 import _lib
    p = pipeline_from({"text": (__import__("pathlib").Path(__file__).resolve().parent.parent
                                / "assets/pipelines/nets/vgg16.pl").read_text()})
    inf = ss._info(p)
    pid = gpu_ctx.pipeline_id(inf.desc)
    gpu_ctx.set_params(v0)
    n = 200_000
    recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nrec = ctypes.c_int64()
    gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 4242, n, recs.data_ptr(),
                                                        offs.data_ptr(), ctypes.byref(nrec)))
    h_recs = np.frombuffer(recs[: nrec.value * 16].cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
    h_offs = offs.cpu().numpy()
    codes = ss.action_codes(inf, h_recs, h_offs)
    assert codes is not None
    d_codes = torch.empty(len(h_recs), dtype=torch.int16, device="cuda")
    gpu_ctx.check(gpu_ctx.lib.ts_encode_codes_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), n,
                                                     d_codes.data_ptr()))
    assert np.array_equal(d_codes.cpu().numpy().view(np.uint16), codes)  # device encoder == host encoder
    depths = np.diff(h_offs).astype(np.uint8)
    for mode in (MODE_EXACT, MODE_FAST):
        a = np.empty(n)
        gpu_ctx.check(gpu_ctx.lib.ts_score_states(gpu_ctx.h, pid, _lib._p(h_recs), _lib._p(h_offs), n, mode,
                                                  _lib._p(a)))
        # device-resident codes (ts_score_states_coded_device)
        d_out = torch.empty(n, dtype=torch.float64, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_score_states_coded_device(gpu_ctx.h, pid, d_codes.data_ptr(), offs.data_ptr(),
                                                               n, len(h_recs), mode, d_out.data_ptr()))
        assert np.array_equal(bits(a), bits(d_out.cpu().numpy())), mode
        # many small chunks alternate between the two scoring lanes (FAST):
        # every chunk must own its offsets and scratch
        for chunk, step in ((None, None), ("50000", None), ("20000", "45000"), ("4096", "6000")):
            if chunk:
                os.environ["TS_CODED_CHUNK"] = chunk
            if step:
                os.environ["TS_CODED_STEP"] = step
            b = np.empty(n)
            try:
                gpu_ctx.check(gpu_ctx.lib.ts_score_states_coded(gpu_ctx.h, pid, _lib._p(codes), _lib._p(depths),
                                                                n, mode, _lib._p(b)))
            finally:
                os.environ.pop("TS_CODED_CHUNK", None)
                os.environ.pop("TS_CODED_STEP", None)
            assert np.array_equal(bits(a), bits(b)), (mode, chunk, step)
    bad = codes.copy()
    bad[5] = 0xF800  # reserved bits set
    b = np.empty(n)
    rc = gpu_ctx.lib.ts_score_states_coded(gpu_ctx.h, pid, _lib._p(bad), _lib._p(depths), n, MODE_FAST,
                                           _lib._p(b))
    assert rc != 0


def test_exact_leg_bit_identical_to_reference(state_sets, v0, golden, greedy_golden):
    """With glibc 2.39's exp and tanh restated on the device
    (csrc/ts_glibc_math.cuh, TS_GLIBC_MATH), the exact leg reproduces the
    reference's Cython kernel + math.exp BIT FOR BIT: V of every golden
    state, backend.lstm_forward's raw on the golden inputs, and the fused
    greedy's predicted V of the final schedule on all 14 pipelines - so
    greedy/beam identity holds by construction, not by tolerance."""
    from paper_2011_14486_b200.backend import lstm_forward
    for name, z in state_sets.items():
        p = pipeline_from(z)
        got = predict_states(v0, product_states(p, z["keys"]), mode=MODE_EXACT)
        assert np.array_equal(bits(got), bits(z["values"])), name
    zf = np.load(golden / "lstm_forward.npz")
    raw = lstm_forward(zf["X"], v0.Wx, v0.Wh, v0.b, v0.w, v0.b_out)
    assert np.array_equal(bits(raw), bits(zf["raw"]))
    for key, g in greedy_golden.items():
        s, visited, v = greedy_schedule_gpu(pipeline_from(g), v0, return_value=True)
        assert [d.render() for d in s.decisions] == g["schedule"], key
        assert v == float.fromhex(g["predicted"]), key


@pytest.mark.parametrize("net", ["vgg16", "resnet18"])
def test_exact_leg_bitwise_on_device_generated_states(gpu_ctx, v0_path, v0, net):
    """1,000 device-generated random partial states per network: the exact
    leg's V (device-resident call) equals the oracle's (C restatement of the
    Cython kernel over libm exp/tanh, pinned to the reference's goldens) bit
    for bit."""
    import ctypes
    import pathlib
    import torch
    p = pipeline_from({"text": (pathlib.Path(__file__).resolve().parent.parent / "assets" / "pipelines" / "nets"
                                / f"{net}.pl").read_text()})
    inf = ss._info(p)
    n = 1000
    with gpu_ctx.lock:
        gpu_ctx.set_params(v0)
        pid = gpu_ctx.pipeline_id(inf.desc)
        recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
        offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        nrec = ctypes.c_int64()
        gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 2024, n, recs.data_ptr(),
                                                            offs.data_ptr(), ctypes.byref(nrec)))
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), n,
                                                         nrec.value, MODE_EXACT, out.data_ptr()))
        got = out.cpu().numpy()
    hr = np.frombuffer(recs[: nrec.value * 16].cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
    ho = offs.cpu().numpy()
    decs = [[O.as_act(inf.decode(k, r)) for k, r in enumerate(hr[ho[i]:ho[i + 1]])] for i in range(n)]
    want = O.values(oracle_params(v0_path), O.Pipe(p), decs)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("key", ["assets/pipelines/nets/crp2d.pl", "assets/pipelines/nets/vgg16.pl"])
def test_greedy_stats_distinct_rows(greedy_golden, v0, key):
    """ts_greedy_stats after the one-kernel greedy layers (distinct children
    rows from the layers' row hashes, k_greedy_distinct) equals a bitwise
    count: along the golden schedule, every layer's children featurized and
    normalized on the device (featurize_states), distinct new rows counted
    in numpy; visited equals the candidate total."""
    import ctypes
    from paper_2011_14486_b200.featurizer import featurize_states
    g = greedy_golden[key]
    p = pipeline_from(g)
    s, visited = greedy_schedule_gpu(p, v0)
    ctx = _lib.context(0)
    vis, distinct = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.ts_greedy_stats(ctx.h, ctypes.byref(vis), ctypes.byref(distinct)))
    T = ss._info(p).T
    want, total = 0, 0
    st = ss.initial_state(p)
    for i, r in enumerate(g["schedule"]):
        kids = [ss.child_state(st, a) for a in ss.candidate_actions(st)]
        total += len(kids)
        rows = [m[T - 1 - i].tobytes() for m in featurize_states(kids, params=v0, normalized=True)]
        want += len(set(rows))
        st = ss.apply(st, ss.parse_layer_schedule(r))
    assert vis.value == visited == total == g["visited"]
    assert distinct.value == want


def test_exact_sweep_kernels_agree_bitwise(gpu_ctx, v0):
    """The exact sweep's two-states-per-warp kernel (k_score_exact32xn<2>,
    depth-sorted pairs, batches >= 4,096) equals the one-state-per-warp
    kernel (k_score_exact32, TS_EXACT_X1) bit for bit on 20,000
    device-generated VGG-16 and ResNet-18 states (ragged depths, odd count:
    the last warp holds one state)."""
    import ctypes
    import os
    import pathlib
    import torch
    for net in ("vgg16", "resnet18"):
        p = pipeline_from({"text": (pathlib.Path(__file__).resolve().parent.parent / "assets" / "pipelines"
                                    / "nets" / f"{net}.pl").read_text()})
        inf = ss._info(p)
        n = 20_001
        with gpu_ctx.lock:
            gpu_ctx.set_params(v0)
            pid = gpu_ctx.pipeline_id(inf.desc)
            recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
            offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            nrec = ctypes.c_int64()
            gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 31337, n, recs.data_ptr(),
                                                                offs.data_ptr(), ctypes.byref(nrec)))
            got = {}
            for x1 in (False, True):
                if x1:
                    os.environ["TS_EXACT_X1"] = "1"
                try:
                    o = torch.empty(n, dtype=torch.float64, device="cuda")
                    gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(),
                                                                     offs.data_ptr(), n, nrec.value, MODE_EXACT,
                                                                     o.data_ptr()))
                    got[x1] = o.cpu().numpy()
                finally:
                    os.environ.pop("TS_EXACT_X1", None)
        assert np.all(got[False] > 0)
        assert np.array_equal(bits(got[False]), bits(got[True])), net


def test_host_wire_paths_multi_chunk_bitwise(gpu_ctx, v0):
    """The host-buffer paths score a large batch in chunks whose offsets are
    absolute (ts_score_states, ts_score_states_packed: the exact leg's rows
    are indexed from each chunk's first record) or chunk-local
    (ts_score_states_coded): 300,000 device-generated VGG-16 states - five
    or more chunks each - equal the device-resident call bit for bit in
    both legs."""
    import ctypes
    import pathlib
    import torch
    p = pipeline_from({"text": (pathlib.Path(__file__).resolve().parent.parent
                                / "assets/pipelines/nets/vgg16.pl").read_text()})
    inf = ss._info(p)
    n = 300_000
    with gpu_ctx.lock:
        gpu_ctx.set_params(v0)
        pid = gpu_ctx.pipeline_id(inf.desc)
        recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
        offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        nrec = ctypes.c_int64()
        gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 99, n, recs.data_ptr(),
                                                            offs.data_ptr(), ctypes.byref(nrec)))
        h_recs = np.frombuffer(recs[: nrec.value * 16].cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
        h_offs = offs.cpu().numpy()
        depths = np.diff(h_offs).astype(np.uint8)
        packed = _lib.pack_records(h_recs)
        codes = ss.action_codes(inf, h_recs, h_offs)
        assert packed is not None and codes is not None
        for mode in (MODE_EXACT, MODE_FAST):
            d = torch.empty(n, dtype=torch.float64, device="cuda")
            gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), n,
                                                             nrec.value, mode, d.data_ptr()))
            want = bits(d.cpu().numpy())
            for name, call in (
                    ("records", lambda o: gpu_ctx.lib.ts_score_states(gpu_ctx.h, pid, _lib._p(h_recs),
                                                                      _lib._p(h_offs), n, mode, _lib._p(o))),
                    ("packed", lambda o: gpu_ctx.lib.ts_score_states_packed(gpu_ctx.h, pid, _lib._p(packed),
                                                                            _lib._p(depths), n, mode, _lib._p(o))),
                    ("coded", lambda o: gpu_ctx.lib.ts_score_states_coded(gpu_ctx.h, pid, _lib._p(codes),
                                                                          _lib._p(depths), n, mode, _lib._p(o)))):
                o = np.empty(n)
                gpu_ctx.check(call(o))
                assert np.array_equal(bits(o), want), (name, mode)
