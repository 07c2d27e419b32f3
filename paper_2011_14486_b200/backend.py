"""Kernel seam (backend.py:15-29) with a `cuda` backend.

The reference selects its recurrent kernels here at import time and calls
them through the module (`backend.lstm_forward`, value_model.py:116;
`backend.lstm_forward_cached` / `backend.lstm_backward`, :197, :202).  The
three functions below keep those signatures and run on the B200:

  lstm_forward(X, Wx, Wh, b, w, b_out) -> raw
      exact fp64 LSTM (ts_lstm_forward; the operation order of
      _recurrent_cy.pyx:38-65)
  lstm_forward_cached(X, Wx, Wh, b, w, b_out) -> (raw, cache)
      raw as above; `cache` is an opaque handle holding the batch and the
      weights it was computed with (_recurrent_np.py:38-59 keeps per-timestep
      activations instead - the device recomputes them, so they never cross
      the boundary)
  lstm_backward(X, Wx, Wh, w, cache, d_raw) -> (dWx, dWh, db, dw, db_out)
      fp64 forward + BPTT + weight gradients on the device
      (ts_lstm_backward; _recurrent_np.py:62-96)

There is no CPU fallback: without the sm_100a library or a B200 every call
raises.  INTEGRATION.md level 2 shows how the unmodified reference is
switched onto this module.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

BACKEND = "cuda"


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _batch(X):
    X = _f64(X)
    if X.ndim != 3:
        raise ValueError("X must be [B, T, F]")
    return X


def lstm_forward(X, Wx, Wh, b, w, b_out, mode: int = _lib.MODE_EXACT, device=None):
    X = _batch(X)
    B, T, F = X.shape
    arrs = [_f64(a) for a in (Wx, Wh, b, w)]
    H = arrs[3].shape[0]
    raw = np.empty(B)
    ctx = _lib.context(device)
    with ctx.lock:
        ctx.check(ctx.lib.ts_lstm_forward(ctx.h, _lib._p(X), B, T, F, _lib._p(arrs[0]),
                                          _lib._p(arrs[1]), _lib._p(arrs[2]), _lib._p(arrs[3]),
                                          H, float(b_out), int(mode), _lib._p(raw)))
    return raw


@dataclass(frozen=True)
class LstmCache:
    """Opaque forward cache: what lstm_backward needs beyond its arguments."""

    X: np.ndarray
    b: np.ndarray
    b_out: float
    device: object = None


def lstm_forward_cached(X, Wx, Wh, b, w, b_out, device=None):
    X = _batch(X)
    raw = lstm_forward(X, Wx, Wh, b, w, b_out, device=device)
    return raw, LstmCache(X, _f64(b).copy(), float(b_out), device)


def lstm_backward(X, Wx, Wh, w, cache, d_raw):
    if not isinstance(cache, LstmCache):
        raise TypeError("cache must come from this backend's lstm_forward_cached")
    X = _batch(X)
    if X.shape != cache.X.shape or not np.array_equal(X, cache.X):
        raise ValueError("lstm_backward: X differs from the cached forward batch")
    B, T, F = X.shape
    Wx, Wh, w = _f64(Wx), _f64(Wh), _f64(w)
    H = w.shape[0]
    G = 4 * H
    d_raw = _f64(d_raw)
    if d_raw.shape != (B,):
        raise ValueError("d_raw must be [B]")
    n = F * G + H * G + G + H + 1
    g = np.empty(n)
    ctx = _lib.context(cache.device)
    with ctx.lock:
        ctx.check(ctx.lib.ts_lstm_backward(ctx.h, _lib._p(X), B, T, F, _lib._p(Wx), _lib._p(Wh),
                                           _lib._p(cache.b), _lib._p(w), H, cache.b_out,
                                           _lib._p(d_raw), _lib._p(g)))
    o = 0
    dWx = g[o: o + F * G].reshape(F, G).copy()
    o += F * G
    dWh = g[o: o + H * G].reshape(H, G).copy()
    o += H * G
    db = g[o: o + G].copy()
    o += G
    dw = g[o: o + H].copy()
    return dWx, dWh, db, dw, float(g[-1])
