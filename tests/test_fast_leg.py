"""The tensor-core (FAST) leg at depth and outside v0's operand range.

* FAST against EXACT on 1e5 device-generated states of every benchmark
  network (T = 34 .. 121: the split-fp16 error grows with the number of
  timesteps) and on 4,096 states of every seeded random pipeline; the
  per-network maximum relative error is printed (DESIGN.md §3 records it).
  Bar: 1e-4 relative (BASELINE.json north_star, fp32 leg).
* Range guard: a checkpoint whose normalizer floors a sigma at 1e-6 (what
  the reference's fit_normalizer does for a constant training column,
  featurizer.py:110-132) puts normalized features near 1e6, past fp16's
  65,504.  States with such a feature are rescored on the exact leg (their
  FAST V equals the EXACT V bit for bit), and a pipeline whose unscheduled
  rows leave the range is scored on the exact leg altogether.  Never NaN.
* Normalized rows bit for bit against featurizer.normalize of the golden
  features (IEEE subtract and divide, featurizer.py:136-137).
"""

import ctypes
import pathlib

import numpy as np
import pytest

from helpers import bits, pipeline_from, product_states
from random_pipelines import random_pipeline_text
from paper_2011_14486_b200 import _lib
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.featurizer import Normalizer, featurize_states, normalize
from paper_2011_14486_b200.value_model import MODE_EXACT, MODE_FAST, load

pytestmark = pytest.mark.gpu

FAST_RTOL = 1e-4
NETS = pathlib.Path(__file__).resolve().parent.parent / "assets" / "pipelines" / "nets"


def _device_states(ctx, p, n, seed):
    import torch
    inf = ss._info(p)
    pid = ctx.pipeline_id(inf.desc)
    recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nrec = ctypes.c_int64()
    ctx.check(ctx.lib.ts_generate_states_device(ctx.h, pid, seed, n, recs.data_ptr(), offs.data_ptr(),
                                                ctypes.byref(nrec)))
    return pid, recs, offs, nrec.value


def _score(ctx, pid, recs, offs, n, nrec, mode):
    import torch
    o = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), n, nrec, mode,
                                             o.data_ptr()))
    return o.cpu().numpy()


def _both(ctx, params, p, n, seed):
    with ctx.lock:
        ctx.set_params(params)
        pid, recs, offs, nrec = _device_states(ctx, p, n, seed)
        return (_score(ctx, pid, recs, offs, n, nrec, MODE_EXACT),
                _score(ctx, pid, recs, offs, n, nrec, MODE_FAST), recs, offs)


@pytest.mark.parametrize("net", ["vgg16", "resnet18", "mobilenet_v2", "resnet50"])
def test_fast_vs_exact_at_depth(gpu_ctx, v0_path, net):
    params = load(v0_path)
    p = pi.parse_pipeline((NETS / f"{net}.pl").read_text())
    exact, fast, _, _ = _both(gpu_ctx, params, p, 100_000, 4242)
    assert np.all(np.isfinite(fast)) and np.all(exact > 0)
    rel = np.abs(fast / exact - 1.0)
    print(f"{net}: T={ss._info(p).T} FAST vs EXACT on 1e5 states: max rel {rel.max():.3e}, "
          f"mean {rel.mean():.3e}")
    assert rel.max() <= FAST_RTOL, (net, rel.max())


def test_fast_vs_exact_random_pipelines(gpu_ctx, v0_path):
    params = load(v0_path)
    worst = 0.0
    for seed in list(range(40)) + list(range(1000, 1012)):
        text = random_pipeline_text(seed, big=seed >= 1000)
        p = pi.parse_pipeline(text)
        exact, fast, _, _ = _both(gpu_ctx, params, p, 4096, 9000 + seed)
        assert np.all(np.isfinite(fast)), seed
        rel = np.abs(fast / exact - 1.0)
        worst = max(worst, rel.max())
        assert rel.max() <= FAST_RTOL, (seed, rel.max())
    print(f"random pipelines: FAST vs EXACT max rel {worst:.3e} (52 pipelines x 4096 states)")


def _floored(params, k, mean):
    """params with normalizer sigma[k] floored at 1e-6 and mean[k] = mean."""
    q = params.copy()
    m = params.normalizer.mean.copy()
    s = params.normalizer.std.copy()
    m[k] = mean
    s[k] = 1e-6
    q.normalizer = Normalizer(m, s)
    return q


def test_range_guard_rescues_out_of_range_states(gpu_ctx, v0_path):
    """sigma[9] (log2 vectorize width) floored with mean 0: unscheduled and
    unvectorized rows stay at 0, every vectorized row normalizes to 3e6.
    Those states go through the exact leg (bit-identical V), the rest stay
    within the FAST bar; nothing is NaN or infinite."""
    params = _floored(load(v0_path), 9, 0.0)
    p = pi.parse_pipeline((NETS / "vgg16.pl").read_text())
    n = 50_000
    exact, fast, recs, offs = _both(gpu_ctx, params, p, n, 31337)
    assert np.all(np.isfinite(fast)) and np.all(np.isfinite(exact))
    rec = np.frombuffer(recs.cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
    o = offs.cpu().numpy()
    vec = rec["vec"][: o[-1]] > 1
    flagged = np.add.reduceat(vec.astype(np.int64), o[:-1]) > 0
    assert 0.1 < flagged.mean() < 0.99, flagged.mean()  # both kinds present
    assert np.array_equal(bits(fast[flagged]), bits(exact[flagged]))
    rel = np.abs(fast[~flagged] / exact[~flagged] - 1.0)
    assert rel.max() <= FAST_RTOL, rel.max()


def test_range_guard_pipeline_outside_range(gpu_ctx, v0_path):
    """sigma[8] (the 'scheduled' indicator) floored with mean 1: every
    unscheduled row normalizes to -1e6, so the pipeline's constant rows are
    outside the operand range and FAST scores it on the exact leg."""
    params = _floored(load(v0_path), 8, 1.0)
    p = pi.parse_pipeline((NETS / "vgg16.pl").read_text())
    exact, fast, _, _ = _both(gpu_ctx, params, p, 20_000, 555)
    assert np.all(np.isfinite(fast))
    assert np.array_equal(bits(fast), bits(exact))
    # the unmodified checkpoint goes back to the tensor cores afterwards
    v0 = load(v0_path)
    exact2, fast2, _, _ = _both(gpu_ctx, v0, p, 20_000, 555)
    assert not np.array_equal(bits(fast2), bits(exact2))
    assert np.abs(fast2 / exact2 - 1).max() <= FAST_RTOL


def test_range_guard_through_the_coded_wire_path(gpu_ctx, v0_path):
    """predict_states with a large batch travels as 16-bit action codes in
    chunks over two scoring lanes; the guard runs per chunk."""
    from paper_2011_14486_b200.value_model import predict_states
    params = _floored(load(v0_path), 9, 0.0)
    z = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "states_vgg16.npz")
    p = pipeline_from({"text": str(z["text"])})
    states = product_states(p, z["keys"]) * 700
    fast = predict_states(params, states, mode=MODE_FAST)
    exact = predict_states(params, states[: len(z["keys"])], mode=MODE_EXACT)
    assert np.all(np.isfinite(fast))
    rel = np.abs(fast / np.tile(exact, 700) - 1)
    assert rel.max() <= FAST_RTOL


def test_normalized_rows_bitwise(state_sets, v0_path):
    params = load(v0_path)
    for name, z in state_sets.items():
        p = pipeline_from(z)
        got = np.stack(featurize_states(product_states(p, z["keys"]), params=params, normalized=True))
        want = np.stack([normalize(params.normalizer, f) for f in z["features"]])
        assert np.array_equal(bits(got), bits(want)), name
