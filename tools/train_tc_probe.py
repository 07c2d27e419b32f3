"""Timing probe for the training kernels (mode tcf/tc/exact) on a synthetic
VGG-16-shaped dataset: B sequences of T = 34 timesteps, random normalized
rows.  Prints ms per gradient call per mode."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2011_14486_b200 import _lib  # noqa: E402
from paper_2011_14486_b200.trainer import DeviceGradients, flat_params  # noqa: E402
from paper_2011_14486_b200.value_model import load  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
T = 34
params = load("tests/golden/v0.ckpt")
rng = np.random.default_rng(0)
N = B
X = rng.normal(size=(N, T, 16))
Tl = np.full(N, T, dtype=np.int32)
logt = rng.normal(5, 2, size=N)
ctx = _lib.context(0)
dev = DeviceGradients(ctx, X, Tl, logt, 32)
dev.set_params(flat_params(params))
gb = torch.zeros(dev.n_params, dtype=torch.float64, device="cuda")
idx = np.arange(B, dtype=np.int32)
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["exact", "tc", "tcf"]
for mode in modes:
    dev.set_mode(mode)
    for _ in range(3):
        dev.grads(idx, B, params.target_scale, gb.data_ptr())
    dev.sync()
    t0 = time.perf_counter()
    for _ in range(10):
        dev.grads(idx, B, params.target_scale, gb.data_ptr())
    dev.sync()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    print(f"{mode}: B={B} {ms:.3f} ms per gradient, {B / ms * 1e3 / 1e6:.2f} M samples/s")
