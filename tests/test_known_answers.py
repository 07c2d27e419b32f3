"""Known answers from the reference SPEC (SPEC.md:100, :255-257, :264-266,
:397, :598-599) through the product's device path."""

import math

import numpy as np
import pytest

from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss

T1 = "pipeline t1_scale\nbuffer src dims 64 elem 4\nstage scale dims x:64 flops 2 output\n  in src map x*1+1\n"
T2 = ("pipeline t2_stencil\nbuffer src dims 66 elem 4\nstage pre dims x:66 flops 1\n  in src map x*1+1\n"
      "stage blur dims x:64 flops 3 output\n  in pre map x*1+3\n")


def test_intrinsic_integers_spec_100():
    """points 64, flops 128, input 256, output 256."""
    d = pi.descriptor(pi.parse_pipeline(T1))
    w = d[4:4 + 48]
    assert (w[13], w[14], w[15], w[16]) == (64, 128, 256, 256)


@pytest.mark.gpu
def test_benchmark_known_answers_spec_264():
    """Default schedule 2432.000; vectorized 2320.000."""
    from paper_2011_14486_b200.cost_oracle import MachineModel, benchmark, format_millis
    p = pi.parse_pipeline(T1)
    s0 = ss.initial_state(p)
    plain = ss.apply(s0, ss.LayerSchedule("scale", (), ("x",)))
    vec = ss.apply(s0, ss.LayerSchedule("scale", (), ("x",), 8))
    par = ss.apply(s0, ss.LayerSchedule("scale", (), ("x",), 1, True))
    assert format_millis(benchmark(plain).total_millis) == "2432.000"
    assert format_millis(benchmark(vec).total_millis) == "2320.000"
    assert benchmark(par).total_millis > benchmark(plain).total_millis  # overhead dominates


@pytest.mark.gpu
def test_stencil_recompute_feature_spec_257():
    """b split x by 8, pre at b's outer loop: invocations 8, region 10,
    recompute 80/66 - as features 13 and 15."""
    from paper_2011_14486_b200.featurizer import featurize_states
    p = pi.parse_pipeline(T2)
    s = ss.apply(ss.initial_state(p), ss.LayerSchedule("blur", (("x", 8),), ("xo", "xi")))
    s = ss.apply(s, ss.LayerSchedule("pre", (), ("x",), 1, False, ("blur", 0)))
    f = featurize_states([s])[0]
    row = f[0]  # topological position 0 = pre
    assert row[8 + 5] == math.log2(80 / 66)
    assert row[8 + 7] == math.log2(1 + 8)
    assert row[8 + 4] == 1.0  # depth


@pytest.mark.gpu
def test_finite_difference_gradient_check_spec_397(v0_path, golden):
    """Every checked coordinate of the device gradient matches central
    differences (h = 1e-4) of the device loss within 1e-4 relative."""
    from paper_2011_14486_b200 import _lib
    from paper_2011_14486_b200.featurizer import featurize_states, normalize
    from paper_2011_14486_b200.trainer import DeviceGradients, flat_params
    from paper_2011_14486_b200.value_model import load
    import json
    g = json.loads((golden / "train_v0.json").read_text())
    pipes = {n: pi.parse_pipeline(t) for n, t in g["pipelines"].items()}
    data = [(ss.state_from_key(pipes[k.split("/", 1)[0]], k), float.fromhex(t))
            for k, t in list(zip(g["keys"], g["targets"]))[:24]]
    params = load(v0_path)
    mats = featurize_states([s for s, _ in data])
    T = np.array([m.shape[0] for m in mats], dtype=np.int32)
    X = np.zeros((len(mats), T.max(), 16))
    for i, m in enumerate(mats):
        X[i, : len(m)] = normalize(params.normalizer, m)
    logt = np.log([t for _, t in data])
    dev = DeviceGradients(_lib.context(0), X, T, logt, params.hidden)
    base = flat_params(params)
    batch = np.argsort(T, kind="stable").astype(np.int32)
    import torch
    gb = torch.zeros(dev.n_params, dtype=torch.float64, device="cuda")
    dev.set_params(base)
    dev.grads(batch, len(batch), params.target_scale, gb.data_ptr())
    dev.sync()
    grad = gb.cpu().numpy()

    def loss(flat):
        dev.set_params(flat)
        raw = dev.forward(batch)
        err = raw + params.target_scale - logt[batch]
        return float(err @ err) / len(batch)

    rng = np.random.default_rng(0)
    n_wx, n_wh = 16 * 128, 32 * 128
    picks = list(rng.choice(n_wx, 5, replace=False)) + list(n_wx + rng.choice(n_wh, 5, replace=False))
    picks += list(n_wx + n_wh + rng.choice(128, 5, replace=False)) + [n_wx + n_wh + 128 + 3, dev.n_params - 1]
    h = 1e-4
    for i in picks:
        e = np.zeros_like(base)
        e[i] = h
        fd = (loss(base + e) - loss(base - e)) / (2 * h)
        assert abs(fd - grad[i]) <= 1e-4 * max(abs(fd), abs(grad[i]), 1e-8), (i, fd, grad[i])
