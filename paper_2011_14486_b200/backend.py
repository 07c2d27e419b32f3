"""Kernel seam (backend.py:15-29) with a `cuda` backend.

`lstm_forward(X, Wx, Wh, b, w, b_out) -> raw` keeps the reference signature
and runs the exact fp64 LSTM kernel on the B200 (same operation order as
_recurrent_cy.pyx:38-65).  There is no CPU fallback: without the sm_100a
library or a B200 the call raises.
"""

from __future__ import annotations

import numpy as np

from . import _lib

BACKEND = "cuda"


def lstm_forward(X, Wx, Wh, b, w, b_out, mode: int = _lib.MODE_EXACT, device=None):
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim != 3:
        raise ValueError("X must be [B, T, F]")
    B, T, F = X.shape
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (Wx, Wh, b, w)]
    H = arrs[3].shape[0]
    raw = np.empty(B)
    ctx = _lib.context(device)
    with ctx.lock:
        ctx.check(ctx.lib.ts_lstm_forward(ctx.h, _lib._p(X), B, T, F, _lib._p(arrs[0]),
                                          _lib._p(arrs[1]), _lib._p(arrs[2]), _lib._p(arrs[3]),
                                          H, float(b_out), int(mode), _lib._p(raw)))
    return raw
