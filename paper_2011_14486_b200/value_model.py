"""Value model on the B200: parameters, checkpoints and batched V(s).

`predict_states` (value_model.py:129-155) is the V-callable behind
`search.model_value`.  Every state goes through one device pass -
featurize (bit-exact) -> normalize -> LSTM -> exp - so results are
independent of `jobs`, batch size and chunking (the reference's
EVAL_CHUNK guarantee, value_model.py:33).  Two precisions:

  MODE_EXACT  fp64 in the Cython kernel's operation order
              (_recurrent_cy.pyx:38-65); used by greedy/beam/learner parity
  MODE_FAST   tcgen05 tensor-core path, fp32-accurate (|dV|/V <= 1e-4)

Checkpoints use the reference's TSVM v1 layout (value_model.py:296-376).
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CheckpointError, PipelineError
from .featurizer import FEATURE_WIDTH, Normalizer
from .schedule_space import action_codes, encode_states

INPUT_DIM = FEATURE_WIDTH
PACKED_MIN = 4096  # batches at least this large travel in the 8-byte wire format
MODE_EXACT = _lib.MODE_EXACT
MODE_FAST = _lib.MODE_FAST


@dataclass
class ValueModelParams:
    hidden: int
    Wx: np.ndarray
    Wh: np.ndarray
    b: np.ndarray
    w: np.ndarray
    b_out: float
    target_scale: float
    normalizer: Normalizer

    def copy(self):
        return ValueModelParams(self.hidden, self.Wx.copy(), self.Wh.copy(), self.b.copy(),
                                self.w.copy(), self.b_out, self.target_scale, self.normalizer)

    def __eq__(self, other):
        return (isinstance(other, ValueModelParams) and self.hidden == other.hidden
                and all(np.array_equal(getattr(self, k), getattr(other, k))
                        for k in ("Wx", "Wh", "b", "w"))
                and self.b_out == other.b_out and self.target_scale == other.target_scale
                and self.normalizer == other.normalizer)


def init_params(seed: int, hidden: int = 32) -> ValueModelParams:
    """Same PCG64 stream and layout as value_model.py:91-107."""
    if hidden < 1:
        raise PipelineError("hidden size must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    s = 1.0 / math.sqrt(hidden)
    b = np.zeros(4 * hidden)
    b[hidden: 2 * hidden] = 1.0
    return ValueModelParams(hidden, rng.uniform(-s, s, (INPUT_DIM, 4 * hidden)),
                            rng.uniform(-s, s, (hidden, 4 * hidden)), b,
                            rng.uniform(-s, s, hidden), 0.0, 0.0,
                            Normalizer(np.zeros(FEATURE_WIDTH), np.ones(FEATURE_WIDTH)))


def predict_states(params, states, jobs: int = 1, mode: int = MODE_EXACT, device=None) -> np.ndarray:
    """V(s) = exp(raw + target_scale) for every state, on the device."""
    out = np.empty(len(states))
    if not states:
        return out
    ctx = _lib.context(device)
    # one critical section from the parameter upload to the last scoring
    # call: a thread sharing the context with other params cannot interleave
    with ctx.lock:
        ctx.set_params(params)
        for inf, idxs, recs, offsets in encode_states(states):
            pid = ctx.pipeline_id(inf.desc)
            vals = np.empty(len(idxs))
            big = len(idxs) >= PACKED_MIN and inf.T < 256
            codes = action_codes(inf, recs, offsets) if big else None
            packed = _lib.pack_records(recs) if big and codes is None else None
            if codes is not None:  # 2 bytes per decision (ts_score_states_coded)
                depths = np.diff(offsets).astype(np.uint8)
                ctx.check(ctx.lib.ts_score_states_coded(ctx.h, pid, _lib._p(codes), _lib._p(depths),
                                                        len(idxs), int(mode), _lib._p(vals)))
            elif packed is not None:  # 8 bytes per decision (ts_score_states_packed)
                depths = np.diff(offsets).astype(np.uint8)
                ctx.check(ctx.lib.ts_score_states_packed(ctx.h, pid, _lib._p(packed), _lib._p(depths),
                                                         len(idxs), int(mode), _lib._p(vals)))
            else:
                ctx.check(ctx.lib.ts_score_states(ctx.h, pid, _lib._p(recs) if len(recs) else None,
                                                  _lib._p(offsets), len(idxs), int(mode),
                                                  _lib._p(vals)))
            out[np.asarray(idxs)] = vals
    return out


def predict(params, state, mode: int = MODE_EXACT) -> float:
    return float(predict_states(params, [state], mode=mode)[0])


def raw_scores(params, X: np.ndarray) -> np.ndarray:
    """Summed per-timestep readouts for a [B, T, 16] batch (value_model.py:114-119)."""
    from .backend import lstm_forward
    return lstm_forward(np.ascontiguousarray(X), params.Wx, params.Wh, params.b, params.w,
                        params.b_out)


# --- checkpoint format (value_model.py:296-306) ----------------------------
MAGIC = b"TSVM"
VERSION = 1


def save(params, path):
    header = json.dumps({"hidden": params.hidden, "b_out": float(params.b_out).hex(),
                         "target_scale": float(params.target_scale).hex()}).encode()
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<II", VERSION, len(header)))
        fh.write(header)
        for arr in (params.Wx, params.Wh, params.b, params.w, params.normalizer.mean,
                    params.normalizer.std):
            fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def load(path) -> ValueModelParams:
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError as e:
        raise CheckpointError(f"cannot read checkpoint: {e}") from None
    if len(data) < 12 or data[:4] != MAGIC:
        raise CheckpointError("not a value-model checkpoint")
    version, hlen = struct.unpack("<II", data[4:12])
    if version != VERSION:
        raise CheckpointError(f"checkpoint version {version} != {VERSION}")
    try:
        header = json.loads(data[12:12 + hlen].decode())
        H = header["hidden"]
        arrays, off = [], 12 + hlen
        for shape in ((INPUT_DIM, 4 * H), (H, 4 * H), (4 * H,), (H,), (FEATURE_WIDTH,),
                      (FEATURE_WIDTH,)):
            n = math.prod(shape)
            chunk = data[off: off + 8 * n]
            if len(chunk) != 8 * n:
                raise CheckpointError("truncated checkpoint")
            arrays.append(np.frombuffer(chunk, dtype="<f8").reshape(shape).copy())
            off += 8 * n
        return ValueModelParams(H, arrays[0], arrays[1], arrays[2], arrays[3],
                                float.fromhex(header["b_out"]),
                                float.fromhex(header["target_scale"]),
                                Normalizer(arrays[4], arrays[5]))
    except CheckpointError:
        raise
    except Exception as e:
        raise CheckpointError(f"corrupt checkpoint: {e}") from None


@dataclass(frozen=True)
class TrainConfig:
    """value_model.py:74-88 (library defaults)."""

    learning_rate: float = 1e-2
    epochs: int = 200
    batch_size: int = 32
    seed: int = 0
    clip_norm: float = 5.0
    holdout_fraction: float = 0.2
    patience: int = 20

    def __post_init__(self):
        if not 0 < self.holdout_fraction < 1:
            raise PipelineError("holdout fraction must be in (0, 1)")
        if min(self.learning_rate, self.epochs, self.batch_size, self.clip_norm,
               self.patience) <= 0:
            raise PipelineError("train config values must be positive")


def train(params, dataset, cfg, device=None, dist=None):
    """value_model.train on the device (see trainer.py)."""
    from .trainer import train as _train
    return _train(params, dataset, cfg, device=device, dist=dist)
