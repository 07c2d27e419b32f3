"""featurize_state on the B200 (featurizer.py:68-107), bit-exact.

The 16-wide rows are produced by the sm_100a kernel `k_featurize_full`
(glibc-log2 port, 256-bit integers, correctly rounded conversions); this
module only moves states in and matrices out.  `Normalizer` /
`fit_normalizer` / `normalize` keep the reference's semantics
(featurizer.py:110-141) - they are elementwise IEEE ops on host arrays the
caller already has.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import PipelineError
from .schedule_space import encode_states

FEATURE_WIDTH = 16
SIGMA_FLOOR = 1e-6
DEFAULT_CACHE_SIZE = 32768  # cost_oracle.MachineModel().cache_size, featurizer.py:75-76


@dataclass(frozen=True)
class Normalizer:
    mean: np.ndarray
    std: np.ndarray

    def __eq__(self, other):
        return (isinstance(other, Normalizer) and np.array_equal(self.mean, other.mean)
                and np.array_equal(self.std, other.std))


def fit_normalizer(dataset) -> Normalizer:
    if not dataset:
        raise PipelineError("cannot fit a normalizer on an empty dataset")
    stacked = np.concatenate([m.reshape(-1, FEATURE_WIDTH) for m in dataset], axis=0)
    return Normalizer(stacked.mean(axis=0), np.maximum(stacked.std(axis=0), SIGMA_FLOOR))


def normalize(nz, mat):
    return (mat - nz.mean) / nz.std


def denormalize(nz, mat):
    return mat * nz.std + nz.mean


_IDENTITY = None


def _identity_params():
    """Featurization needs no weights, but the context computes the shared
    unscheduled rows together with the normalizer; raw features are taken
    from the `normalized=0` path, independent of the uploaded params."""
    global _IDENTITY
    if _IDENTITY is None:
        class _P:  # minimal duck-typed ValueModelParams
            hidden = 32
            Wx = np.zeros((16, 128))
            Wh = np.zeros((32, 128))
            b = np.zeros(128)
            w = np.zeros(32)
            b_out = 0.0
            target_scale = 0.0
            normalizer = Normalizer(np.zeros(16), np.ones(16))
        _IDENTITY = _P()
    return _IDENTITY


def featurize_states(states, cache_size=None, params=None, normalized=False, device=None):
    """[n][T][16] f64 feature matrices for same-length states (device)."""
    if cache_size not in (None, DEFAULT_CACHE_SIZE):
        raise PipelineError("only the default cache size (32768) is featurized on device")
    ctx = _lib.context(device)
    out = [None] * len(states)
    with ctx.lock:  # params upload and the calls that normalize with them
        if params is None:
            if normalized:
                raise PipelineError("normalized features need params")
            if ctx._params_key is None:
                ctx.set_params(_identity_params())
        else:
            ctx.set_params(params)
        for inf, idxs, recs, offsets in encode_states(states):
            pid = ctx.pipeline_id(inf.desc)
            buf = np.empty((len(idxs), inf.T, FEATURE_WIDTH), dtype=np.float64)
            ctx.check(ctx.lib.ts_featurize_states(
                ctx.h, pid, _lib._p(recs) if len(recs) else None, _lib._p(offsets), len(idxs),
                1 if normalized else 0, _lib._p(buf)))
            for j, i in enumerate(idxs):
                out[i] = buf[j]
    return out


def featurize_state(s, cache_size=None):
    """featurizer.featurize_state: cached on the state like the reference
    (featurizer.py:72-73, :104-106)."""
    cache = getattr(s, "_cache", None)
    if isinstance(cache, dict) and "features" in cache:
        return cache["features"]
    mat = featurize_states([s], cache_size)[0]
    mat.setflags(write=False)
    if isinstance(cache, dict):
        cache["features"] = mat
    return mat
