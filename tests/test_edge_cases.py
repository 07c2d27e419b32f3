"""Edge cases of the boundary: empty and ragged batches, the empty prefix
and complete states, illegal records, envelope limits, error mapping."""

import numpy as np
import pytest

import oracle as O
from helpers import bits, oracle_params, pipeline_from
from paper_2011_14486_b200 import _lib
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.errors import IllegalActionError, PipelineError

T1 = "pipeline one\nbuffer src dims 64 elem 4\nstage s dims x:64 flops 2 output\n  in src map x*1+1\n"


def test_descriptor_rejects_outside_envelope():
    wide = ("pipeline wide\nbuffer b dims 2x2x2x2x2 elem 4\n"
            "stage s dims a:2,b:2,c:2,d:2,e:2 flops 1 output\n  in b map a*1+1, b*1+1, c*1+1, d*1+1, e*1+1\n")
    with pytest.raises(PipelineError):
        pi.descriptor(pi.parse_pipeline(wide))


def test_encode_rejects_illegal_structure(greedy_golden):
    p = pipeline_from(greedy_golden["ref:pipelines/toys/t3_chain.pl"])
    s = ss.initial_state(p)
    with pytest.raises(IllegalActionError):
        ss.apply(s, ss.LayerSchedule("pool", (("x", 8),), ("x",)))      # order misses xo/xi
    with pytest.raises(IllegalActionError):
        ss.apply(s, ss.LayerSchedule("pool", (("q", 8),), ("x",)))      # unknown dim
    with pytest.raises(IllegalActionError):
        ss.apply(s, ss.LayerSchedule("pool", (), ("x",), 1, False, ("relu", 0)))  # no consumer


def test_complete_state_candidates_raise(greedy_golden):
    g = greedy_golden["ref:pipelines/toys/t1_scale.pl"]
    p = pipeline_from(g)
    s = ss.initial_state(p)
    s = ss.apply(s, ss.candidate_actions(s)[0])
    assert s.is_complete
    with pytest.raises(IllegalActionError):
        ss.candidate_actions(s)


@pytest.mark.gpu
def test_empty_batch_and_depth_extremes(v0_path, greedy_golden):
    from paper_2011_14486_b200.featurizer import featurize_states
    from paper_2011_14486_b200.value_model import MODE_EXACT, MODE_FAST, load, predict_states
    v0 = load(v0_path)
    assert len(predict_states(v0, [])) == 0
    p = pipeline_from(greedy_golden["assets/pipelines/nets/vgg16.pl"])
    P = O.Pipe(p)
    empty = ss.initial_state(p)                       # d = 0: all rows unscheduled
    full = O.random_partial(P, 3)
    while len(full) < len(P.topo):                    # complete the state: d = T
        full.append(O.candidates(P, full)[0])
    complete = ss.state_from_decisions(p, full)
    states = [empty, complete, empty, complete]
    want = O.values(oracle_params(v0_path), P, [[], full, [], full])
    assert np.array_equal(bits(predict_states(v0, states, mode=MODE_EXACT)), bits(want))  # exact leg: bitwise
    np.testing.assert_allclose(predict_states(v0, states, mode=MODE_FAST), want, rtol=1e-4)
    f = featurize_states([empty, complete])
    assert np.array_equal(bits(f[0]), bits(O.features(P, [])))
    assert np.array_equal(bits(f[1]), bits(O.features(P, full)))


@pytest.mark.gpu
def test_ragged_multi_pipeline_batch(state_sets, v0_path):
    """One predict_states call mixing pipelines of different lengths keeps
    every state's value and the input order."""
    from paper_2011_14486_b200.value_model import load, predict_states
    v0 = load(v0_path)
    states, want = [], []
    for name in ("t1_scale", "t5_diamond", "p12_deep", "vgg16"):
        z = state_sets[name]
        p = pipeline_from(z)
        for k, v in zip(z["keys"][:5], z["values"][:5]):
            states.append(ss.state_from_key(p, str(k)))
            want.append(v)
    order = np.random.default_rng(0).permutation(len(states))
    got = predict_states(v0, [states[i] for i in order])
    assert np.array_equal(bits(got), bits(np.array(want)[order]))


@pytest.mark.gpu
def test_device_rejects_illegal_records(gpu_ctx, greedy_golden, v0_path):
    """A record anchoring at a loop level that does not exist raises
    IllegalActionError through the device status word."""
    from paper_2011_14486_b200.value_model import load
    p = pipeline_from(greedy_golden["ref:pipelines/toys/t3_chain.pl"])
    inf = ss._info(p)
    gpu_ctx.set_params(load(v0_path))
    pid = gpu_ctx.pipeline_id(inf.desc)
    s = ss.initial_state(p)
    a = ss.candidate_actions(s)[0]
    rec0 = np.frombuffer(inf.encode(0, a), dtype=_lib.DECISION_DTYPE).copy()
    rec1 = np.frombuffer(inf.encode(1, ss.candidate_actions(ss.child_state(s, a))[0]),
                         dtype=_lib.DECISION_DTYPE).copy()
    rec1["anchor"] = 7  # level 7 of a 1-loop nest
    recs = np.concatenate([rec0, rec1])
    offs = np.array([0, 2], dtype=np.int64)
    out = np.empty(1)
    with pytest.raises(IllegalActionError):
        gpu_ctx.check(gpu_ctx.lib.ts_score_states(gpu_ctx.h, pid, _lib._p(recs), _lib._p(offs), 1, 0,
                                                  _lib._p(out)))
    # the context stays usable afterwards
    ok = np.concatenate([rec0])
    gpu_ctx.check(gpu_ctx.lib.ts_score_states(gpu_ctx.h, pid, _lib._p(ok),
                                              _lib._p(np.array([0, 1], dtype=np.int64)), 1, 0,
                                              _lib._p(out)))
    assert out[0] > 0


@pytest.mark.gpu
def test_single_stage_pipeline_greedy(v0_path):
    from paper_2011_14486_b200.search import greedy_schedule_gpu
    from paper_2011_14486_b200.value_model import load
    p = pi.parse_pipeline(T1)
    s, visited = greedy_schedule_gpu(p, load(v0_path))
    P = O.Pipe(p)
    want, wv = O.greedy(P, oracle_params(v0_path))
    assert [d.render() for d in s.decisions] == [a.render() for a in want] and visited == wv


@pytest.mark.gpu
def test_deep_compute_at_levels(v0_path):
    """compute_at below level 2 (legal for hand-written schedules, never
    proposed by candidate_actions): features bit-exact against the oracle,
    V on both legs against the oracle's."""
    from paper_2011_14486_b200.featurizer import featurize_states
    from paper_2011_14486_b200.value_model import MODE_FAST, load, predict_states
    text = ("pipeline deep\nbuffer src dims 66x66 elem 4\n"
            "stage pre dims x:66,y:66 flops 1\n  in src map x*1+1, y*1+1\n"
            "stage blur dims x:64,y:64 flops 3 output\n  in pre map x*1+3, y*1+3\n")
    p = pi.parse_pipeline(text)
    P = O.Pipe(p)
    blur = ss.LayerSchedule("blur", (("x", 8), ("y", 8)), ("xo", "xi", "yo", "yi"))
    states = []
    for lvl in range(4):
        pre = ss.LayerSchedule("pre", (), ("x", "y"), 1, False, ("blur", lvl))
        s = ss.apply(ss.initial_state(p), blur)
        if ss.check_action(s, pre) is None:
            states.append(ss.apply(s, pre))
    assert len(states) >= 3 and any(st.decisions[-1].compute_at[1] == 3 for st in states)
    decs = [[O.as_act(d) for d in st.decisions] for st in states]
    feats = featurize_states(states)
    for f, d in zip(feats, decs):
        assert np.array_equal(bits(f), bits(O.features(P, d)))
    params = load(v0_path)
    want = O.values(oracle_params(v0_path), P, decs)
    assert np.array_equal(bits(predict_states(params, states)), bits(want))
    np.testing.assert_allclose(predict_states(params, states * 2000, mode=MODE_FAST), np.tile(want, 2000),
                               rtol=1e-4)


def test_round_config_rejects_zero_schedules():
    """learner.RoundConfig validates like the reference (learner.py:131-133)."""
    from paper_2011_14486_b200.learner import RoundConfig
    with pytest.raises(PipelineError):
        RoundConfig(schedules_per_pipeline=0)
    assert RoundConfig(schedules_per_pipeline=1).schedules_per_pipeline == 1


@pytest.mark.gpu
def test_beam_rejects_illegal_prefix(v0_path, greedy_golden):
    from paper_2011_14486_b200.search import beam_search_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    g = greedy_golden["ref:pipelines/toys/t3_chain.pl"]
    p = pipeline_from(g)
    # a compute_at level the consumer's nest does not have
    bad = ss.ScheduleState(p, (ss.parse_layer_schedule(g["schedule"][0]),
                               ss.LayerSchedule("relu", (), ("x",), 1, False, ("pool", 7), None)))
    with pytest.raises((IllegalActionError, PipelineError)):
        beam_search_gpu(bad, params, 4)


@pytest.mark.gpu
def test_backend_backward_edge_cases(v0_path):
    """Empty batch, a single timestep, and a cache from another batch."""
    from paper_2011_14486_b200 import backend
    from paper_2011_14486_b200.value_model import load
    p = load(v0_path)
    X0 = np.zeros((0, 5, 16))
    raw, cache = backend.lstm_forward_cached(X0, p.Wx, p.Wh, p.b, p.w, p.b_out)
    assert raw.shape == (0,)
    g = backend.lstm_backward(X0, p.Wx, p.Wh, p.w, cache, np.zeros(0))
    assert all(np.all(np.asarray(x) == 0) for x in g)
    X1 = np.random.default_rng(0).normal(size=(3, 1, 16))
    raw, cache = backend.lstm_forward_cached(X1, p.Wx, p.Wh, p.b, p.w, p.b_out)
    dWx, dWh, db, dw, db_out = backend.lstm_backward(X1, p.Wx, p.Wh, p.w, cache, np.ones(3))
    assert np.all(dWh == 0)  # h_{-1} = 0: no recurrent gradient with one timestep
    assert db_out == 3.0
    with pytest.raises(ValueError):
        backend.lstm_backward(X1 + 1.0, p.Wx, p.Wh, p.w, cache, np.ones(3))
