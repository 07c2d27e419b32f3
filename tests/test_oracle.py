"""The CPU oracle (oracle/oracle.py, oracle/lstm_ref.c) against golden
vectors produced by the unmodified reference (tools/make_golden.py)."""

import math

import numpy as np
import pytest

import oracle as O
from helpers import bits, oracle_decisions, oracle_params, pipeline_from


def test_candidates_match_reference(candidates_golden, greedy_golden):
    for key, walk in candidates_golden.items():
        p = pipeline_from(greedy_golden[key])
        P = O.Pipe(p)
        rng = O.SplitMix(5)
        decisions = []
        for step in walk:
            c = O.candidates(P, decisions)
            assert [a.render() for a in c] == step, (key, len(decisions))
            decisions.append(c[rng.randrange(len(c))])


def test_features_bit_exact(state_sets):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        P = O.Pipe(p)
        n = min(len(z["keys"]), 12)
        for i in range(n):
            got = O.features(P, oracle_decisions(p, z["keys"][i]))
            assert np.array_equal(bits(got), bits(z["features"][i])), (name, i)


def test_random_partial_states_match_reference_walk(state_sets):
    for name, z in state_sets.items():
        p = pipeline_from(z)
        P = O.Pipe(p)
        for i in range(min(4, len(z["seeds"]))):
            d = O.random_partial(P, int(z["seeds"][i]))
            key = p.name + "/" + ";".join(a.render() for a in d)
            assert key == str(z["keys"][i]), (name, i)


def test_values_bit_exact(state_sets, v0_path):
    params = oracle_params(v0_path)
    for name in ("t3_chain", "p12_deep", "vgg16", "resnet18"):
        z = state_sets[name]
        p = pipeline_from(z)
        P = O.Pipe(p)
        n = min(len(z["keys"]), 8)
        got = O.values(params, P, [oracle_decisions(p, k) for k in z["keys"][:n]])
        assert np.array_equal(bits(got), bits(z["values"][:n])), name


def test_lstm_forward_bit_exact(golden, v0_path):
    params = oracle_params(v0_path)
    z = np.load(golden / "lstm_forward.npz")
    raw = O.lstm_forward(z["X"], params["Wx"], params["Wh"], params["b"], params["w"],
                         params["b_out"])
    assert np.array_equal(bits(raw), bits(z["raw"]))


SMALL = ["ref:pipelines/toys/t1_scale.pl", "ref:pipelines/toys/t2_stencil.pl",
         "ref:pipelines/toys/t3_chain.pl", "ref:pipelines/toys/t4_reduce.pl",
         "ref:pipelines/toys/t5_diamond.pl", "ref:pipelines/train/train_matmul.pl"]


@pytest.mark.parametrize("key", SMALL)
def test_greedy_matches_reference(key, greedy_golden, v0_path):
    params = oracle_params(v0_path)
    g = greedy_golden[key]
    P = O.Pipe(pipeline_from(g))
    decisions, visited = O.greedy(P, params)
    assert [a.render() for a in decisions] == g["schedule"]
    assert visited == g["visited"]
    v = O.values(params, P, [decisions])[0]
    assert v.hex() == g["predicted"]


def test_noisy_greedy_matches_reference(noisy_golden, greedy_golden, v0_path):
    params = oracle_params(v0_path)
    key = "ref:pipelines/toys/t3_chain.pl#11"
    g = noisy_golden[key]
    P = O.Pipe(pipeline_from(greedy_golden[key.split("#")[0]]))
    rng = O.SplitMix(11)
    decisions, visited = O.greedy(P, params, 0.25, rng)
    assert [a.render() for a in decisions] == g["schedule"]
    assert visited == g["visited"] and rng.state == g["rng_state"]


def test_checkpoint_reader(v0_path):
    params = oracle_params(v0_path)
    assert params["hidden"] == 32 and params["Wx"].shape == (16, 128)
    assert math.isfinite(params["b_out"]) and params["std"].min() >= 1e-6
