"""beam_search (search.py:115-133) against the unmodified reference's
results (tests/golden/beam.json, tools/make_golden_beam.py): width 1/3/8
from the initial state and width 8 (4 on ResNet-18) from mid-schedule
prefixes, on the toys, p12_deep, crp2d, VGG-16, ResNet-18, MobileNet-v2 and
ResNet-50 (the paper's DNN benchmarks, width 8).  The oracle's
beam is checked against the same fixtures on the small pipelines (CPU);
the fused device beam (ts_beam) and the generic loop over the device
V-callable must both return the reference's schedule."""

import json
import pathlib

import numpy as np
import pytest

import oracle as O
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss

GOLD = pathlib.Path(__file__).resolve().parent / "golden" / "beam.json"


def _cases():
    return json.loads(GOLD.read_text())


def _prefix_state(p, renders):
    return ss.state_from_decisions(p, [ss.parse_layer_schedule(r) for r in renders])


def test_oracle_beam_matches_reference_on_small_pipelines(v0_path):
    params = O.load_checkpoint(v0_path)
    for key, c in _cases().items():
        if "nets/" in key and "crp2d" not in key or "p12_deep" in key:
            continue  # the oracle's Python featurizer: small cases only
        p = pi.parse_pipeline(c["text"])
        P = O.Pipe(p)
        prefix = [O.as_act(ss.parse_layer_schedule(r)) for r in c["prefix"]]
        got = O.beam(P, params, prefix, c["width"])
        assert [a.render() for a in got] == c["schedule"], key


@pytest.mark.gpu
def test_fused_device_beam_matches_reference(v0_path):
    from paper_2011_14486_b200.search import beam_search_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    for key, c in _cases().items():
        p = pi.parse_pipeline(c["text"])
        s, v = beam_search_gpu(_prefix_state(p, c["prefix"]), params, c["width"], return_value=True)
        assert [d.render() for d in s.decisions] == c["schedule"], key
        assert abs(v / float.fromhex(c["predicted"]) - 1) < 1e-12, key


@pytest.mark.gpu
def test_generic_beam_over_device_v_matches_reference(v0_path):
    """search.beam_search with a V-callable that has no fused path (one
    device batch per layer through predict_states)."""
    from paper_2011_14486_b200.search import beam_search, model_value
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    V = model_value(params)
    plain = lambda states: V(states)  # noqa: E731  (no .beam attribute)
    for key, c in _cases().items():
        if "resnet" in key or "mobilenet" in key:
            continue  # the generic loop materializes every child on the host
        p = pi.parse_pipeline(c["text"])
        s = beam_search(_prefix_state(p, c["prefix"]), plain, c["width"])
        assert [d.render() for d in s.decisions] == c["schedule"], key


@pytest.mark.gpu
def test_beam_width_one_is_greedy(v0_path, greedy_golden):
    from paper_2011_14486_b200.search import beam_search_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    for key in ("assets/pipelines/nets/resnet50.pl", "assets/pipelines/nets/mobilenet_v2.pl"):
        g = greedy_golden[key]
        p = pi.parse_pipeline(g["text"])
        s = beam_search_gpu(ss.initial_state(p), params, 1)
        assert [d.render() for d in s.decisions] == g["schedule"], key


@pytest.mark.gpu
def test_beam_edge_cases(v0_path, greedy_golden):
    from paper_2011_14486_b200.errors import PipelineError
    from paper_2011_14486_b200.search import beam_search_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    g = greedy_golden["ref:pipelines/toys/t3_chain.pl"]
    p = pi.parse_pipeline(g["text"])
    with pytest.raises(PipelineError):
        beam_search_gpu(ss.initial_state(p), params, 0)
    full = _prefix_state(p, g["schedule"])
    s = beam_search_gpu(full, params, 8)  # a complete prefix is returned as is
    assert [d.render() for d in s.decisions] == g["schedule"]
    big = beam_search_gpu(ss.initial_state(p), params, 1000)  # width above the child count
    assert len(big.decisions) == len(g["schedule"])
