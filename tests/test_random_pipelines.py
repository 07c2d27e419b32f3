"""Parity on seeded random pipelines (tests/random_pipelines.py) beyond the
checked-in networks: candidate enumeration (native host enumerator vs the
oracle, and the oracle vs the built reference when oracle/_ref is present),
device features, both V legs and the fused greedy vs the oracle."""

import pathlib
import sys

import numpy as np
import pytest

import oracle as O
from helpers import bits
from random_pipelines import random_pipeline_text
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss

SEEDS = range(40)
BIG = range(1000, 1012)  # random_pipeline_text(seed, big=True)


def _texts():
    return [random_pipeline_text(s) for s in SEEDS] + [random_pipeline_text(s, big=True) for s in BIG]
REF = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref"


def _walks(P, n, seed0):
    return [O.random_partial(P, seed0 + k) for k in range(n)]


def test_random_pipeline_candidates_native_vs_oracle():
    for seed, text in enumerate(_texts()):
        p = pi.parse_pipeline(text)
        P = O.Pipe(p)
        for decs in _walks(P, 4, 100 * seed + 1):
            s = ss.initial_state(p)
            for k in range(len(decs)):
                want = [a.render() for a in O.candidates(P, decs[:k])]
                got = [a.render() for a in ss.candidate_actions(s)]
                assert got == want, (seed, k)
                s = ss.apply(s, ss.parse_layer_schedule(decs[k].render()))


def test_random_pipeline_oracle_vs_reference():
    """The oracle against the unmodified reference on the same random
    pipelines (candidates and feature matrices, bit for bit)."""
    if not (REF / "tensched").exists():
        pytest.skip("oracle/_ref (the built reference) is not present")
    sys.path.insert(0, str(REF))
    from tensched.featurizer import featurize_state
    from tensched.pipeline_ir import parse_pipeline as ref_parse
    from tensched.schedule_space import apply as ref_apply
    from tensched.schedule_space import candidate_actions as ref_candidates
    from tensched.schedule_space import initial_state as ref_initial
    for seed, text in enumerate(_texts()):
        P = O.Pipe(pi.parse_pipeline(text))
        rp = ref_parse(text)
        for decs in _walks(P, 3, 100 * seed + 7):
            s = ref_initial(rp)
            for k in range(len(decs)):
                cands = ref_candidates(s)
                assert [a.render() for a in cands] == [a.render() for a in O.candidates(P, decs[:k])], (seed, k)
                s = ref_apply(s, next(a for a in cands if a.render() == decs[k].render()))
            assert np.array_equal(bits(np.asarray(featurize_state(s))), bits(O.features(P, decs))), seed


@pytest.mark.gpu
def test_random_pipeline_device_parity(v0_path):
    from paper_2011_14486_b200.featurizer import featurize_states
    from paper_2011_14486_b200.search import greedy_schedule_gpu
    from paper_2011_14486_b200.value_model import MODE_FAST, load, predict_states
    params = load(v0_path)
    oparams = O.load_checkpoint(v0_path)
    for seed, text in enumerate(_texts()):
        p = pi.parse_pipeline(text)
        P = O.Pipe(p)
        decs = _walks(P, 24, 100 * seed + 3)
        states = [ss.state_from_decisions(p, d) for d in decs]
        for f, d in zip(featurize_states(states), decs):
            assert np.array_equal(bits(f), bits(O.features(P, d))), seed
        want = O.values(oparams, P, decs)
        assert np.array_equal(bits(predict_states(params, states)), bits(want)), seed
        reps = -(-4096 // len(states))  # large enough for the compact wire formats
        np.testing.assert_allclose(predict_states(params, states * reps, mode=MODE_FAST), np.tile(want, reps),
                                   rtol=1e-4)
        s, visited = greedy_schedule_gpu(p, params)
        gw, gv = O.greedy(P, oparams)
        assert [d.render() for d in s.decisions] == [a.render() for a in gw] and visited == gv, seed


@pytest.mark.gpu
def test_random_pipeline_beam_parity(v0_path):
    """The fused device beam (ts_beam) against the oracle's beam_search
    restatement on the random pipelines (widths 2 and 4, from the empty
    prefix and from a two-decision prefix): identical completions, V bit for
    bit (the exact leg ranks them)."""
    from paper_2011_14486_b200.search import beam_search_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    oparams = O.load_checkpoint(v0_path)
    checked = 0
    for seed, text in enumerate(_texts()):
        p = pi.parse_pipeline(text)
        P = O.Pipe(p)
        if len(P.topo) > 12:  # the oracle beam is pure Python
            continue
        for width, plen in ((2, 0), (4, 2)):
            prefix = _walks(P, 1, 7 * seed + width)[0][:plen] if plen else []
            if len(prefix) >= len(P.topo):
                continue
            want = O.beam(P, oparams, prefix, width)
            s, v = beam_search_gpu(ss.state_from_decisions(p, prefix), params, width, return_value=True)
            assert [d.render() for d in s.decisions] == [a.render() for a in want], (seed, width, plen)
            assert np.array_equal(bits(np.array([v])), bits(O.values(oparams, P, [want]))), (seed, width)
            checked += 1
    assert checked >= 20


@pytest.mark.gpu
def test_random_pipeline_noisy_greedy_parity(v0_path):
    """The fused device greedy with noise (epsilon 0.25, the learner's
    rollouts) against the oracle's greedy with its SplitMix stream on every
    random pipeline: identical schedules, visited counts and final rng
    state."""
    from paper_2011_14486_b200.search import NoiseConfig, SearchRng, greedy_schedule_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    oparams = O.load_checkpoint(v0_path)
    for seed, text in enumerate(_texts()):
        p = pi.parse_pipeline(text)
        P = O.Pipe(p)
        rng, orng = SearchRng(1000 + seed), O.SplitMix(1000 + seed)
        s, visited = greedy_schedule_gpu(p, params, NoiseConfig(0.25), rng)
        want, ov = O.greedy(P, oparams, 0.25, orng)
        assert [d.render() for d in s.decisions] == [a.render() for a in want], seed
        assert visited == ov and rng.state == orng.state, seed


@pytest.mark.gpu
def test_random_pipeline_score_children_parity(v0_path):
    """ts_score_children (one layer step for any parent: the parent's rows
    once, each child's new row, dedup, the exact suffix LSTM) against the
    oracle's V of the materialized children, bit for bit, on two random
    prefixes of every random pipeline."""
    from paper_2011_14486_b200.search import score_children
    from paper_2011_14486_b200.value_model import load
    params = load(v0_path)
    oparams = O.load_checkpoint(v0_path)
    for seed, text in enumerate(_texts()):
        p = pi.parse_pipeline(text)
        P = O.Pipe(p)
        for decs in _walks(P, 2, 31 * seed + 5):
            if len(decs) >= len(P.topo):
                decs = decs[:-1]
            s = ss.state_from_decisions(p, decs)
            acts = ss.candidate_actions(s)
            got = score_children(params, s, acts)
            want = O.values(oparams, P, [list(decs) + [O.as_act(a)] for a in acts])
            assert np.array_equal(bits(np.asarray(got)), bits(want)), seed
