"""ts_score_children: one layer step for an arbitrary parent.
V of every child must be bit-identical to predict_states on the materialized
children (same exact leg) and within the exact tolerance of the CPU oracle;
the fused argmin must reproduce the host loop of greedy_schedule
(search.py:97-110) including the noise draws and the rng advance."""

import numpy as np
import pytest

import oracle as O
from helpers import bits, oracle_params, pipeline_from
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.errors import PipelineError
from paper_2011_14486_b200.search import (NoiseConfig, SearchRng, beam_search, model_value,
                                          score_children)
from paper_2011_14486_b200.value_model import load, predict_states

pytestmark = pytest.mark.gpu

NETS = ("assets/pipelines/nets/vgg16.pl", "assets/pipelines/nets/resnet18.pl",
        "assets/pipelines/nets/mobilenet_v2.pl", "ref:pipelines/deep/p12_deep.pl",
        "ref:pipelines/toys/t3_chain.pl")


@pytest.fixture(scope="module")
def v0(v0_path):
    return load(v0_path)


def _parents(p, P, seeds):
    out = [ss.initial_state(p)]
    for seed in seeds:
        d = O.random_partial(P, seed)
        if len(d) < len(p.stages):
            out.append(ss.state_from_decisions(p, d))
    return out


def test_children_values_bit_identical(greedy_golden, v0, v0_path):
    oparams = oracle_params(v0_path)
    for key in NETS:
        p = pipeline_from(greedy_golden[key])
        P = O.Pipe(p)
        for s in _parents(p, P, range(300, 306)):
            acts = ss.candidate_actions(s)
            kids = [ss.child_state(s, a) for a in acts]
            got = score_children(v0, s, acts)
            want = predict_states(v0, kids)
            assert np.array_equal(bits(got), bits(want)), (key, len(s.decisions))
            oracle_v = O.values(oparams, P, [[O.as_act(d) for d in k.decisions] for k in kids[:8]])
            assert np.array_equal(bits(got[:8]), bits(oracle_v))


def test_children_argmin_with_noise(greedy_golden, v0):
    p = pipeline_from(greedy_golden["assets/pipelines/nets/resnet18.pl"])
    P = O.Pipe(p)
    for i, s in enumerate(_parents(p, P, range(400, 404))):
        acts = ss.candidate_actions(s)
        vals = predict_states(v0, [ss.child_state(s, a) for a in acts])
        for eps in (0.0, 0.25):
            host_rng, dev_rng = SearchRng(77 + i), SearchRng(77 + i)
            noisy = [v * (1.0 + host_rng.uniform(-eps, eps)) for v in vals] if eps else list(vals)
            want = min(range(len(noisy)), key=lambda k: (noisy[k], k))
            got, got_v = score_children(v0, s, acts, noise=NoiseConfig(eps), rng=dev_rng, best=True)
            assert got == want and got_v == noisy[want]
            assert dev_rng.state == (host_rng.state if eps else 77 + i)


def test_generic_greedy_and_beam_agree_with_plain_callable(greedy_golden, v0):
    """greedy_schedule over model_value (children through score_children)
    and beam_search over it equal the same searches over a plain
    predict_states callable."""
    p = pipeline_from(greedy_golden["ref:pipelines/deep/p12_deep.pl"])
    plain = lambda states: predict_states(v0, states)  # noqa: E731
    for width in (1, 3):
        a = beam_search(ss.initial_state(p), model_value(v0), width)
        b = beam_search(ss.initial_state(p), plain, width)
        assert a.decisions == b.decisions
    from paper_2011_14486_b200.search import greedy_schedule
    a, va = greedy_schedule(p, model_value(v0))
    b, vb = greedy_schedule(p, plain)
    assert a.decisions == b.decisions and va == vb


def test_illegal_child_rejected(greedy_golden, v0):
    p = pipeline_from(greedy_golden["ref:pipelines/toys/t3_chain.pl"])
    s = ss.initial_state(p)
    acts = ss.candidate_actions(s)
    s1 = ss.child_state(s, acts[0])
    with pytest.raises(PipelineError):
        score_children(v0, s1, acts[:2])  # decisions for the wrong stage


def test_children_deep_parent_long_suffix(v0):
    """ResNet-50 (T = 121) parents one and sixty stages short of complete:
    the child's suffix LSTM stages up to 121 rows plus its per-step readout
    in shared memory (past the 48 KB default), and must still equal
    predict_states on the materialized children bit for bit."""
    from paper_2011_14486_b200.pipeline_ir import parse_pipeline
    import pathlib
    root = pathlib.Path(__file__).resolve().parent.parent
    p = parse_pipeline((root / "assets/pipelines/nets/resnet50.pl").read_text())
    T = len(p.stages)
    s = ss.initial_state(p)
    parents = {}
    for i in range(T - 1):
        acts = ss.candidate_actions(s)
        s = ss.child_state(s, acts[i % len(acts)])
        if len(s.decisions) in (60, T - 1):
            parents[len(s.decisions)] = s
    for depth, s in parents.items():
        acts = ss.candidate_actions(s)
        kids = [ss.child_state(s, a) for a in acts]
        got = score_children(v0, s, acts)
        want = predict_states(v0, kids)
        assert np.array_equal(bits(got), bits(want)), depth
