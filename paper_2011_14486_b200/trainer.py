"""V training on the B200 (value_model.train, value_model.py:241-293).

Same host loop as the reference - the PCG64 holdout split and epoch
permutations (:248-263), minibatches grouped by sequence length, global-norm
clipping at `clip_norm` including b_out (:213-220), plain SGD (:267-271),
plateau halving with restore-best every patience//2 stale epochs, early
stop, and the final metrics of `_eval_split` (:223-238) - with every
gradient computed on the device (ts_train_grads: cached forward + BPTT +
weight-gradient reduction, fp64) and the update applied on the device
(ts_train_apply).  Parameters stay resident between steps.

`mode`: "exact" (default) keeps every gradient in fp64, the reference's
trajectory; "tc" keeps the fp64 forward/BPTT recurrences and computes the
weight-gradient contraction on the tensor cores (3xTF32, fused into BPTT,
ts_train_set_mode(TS_TRAIN_TC)) - gradients within ~1e-5 relative of the
exact ones (tested), not bit-identical.

Data parallel: pass `dist` (an initialised torch.distributed default group).
Each rank takes a contiguous shard of every (length-sorted) global
minibatch, computes its gradient with d_raw divided by the GLOBAL batch size,
and the gradient buffer (a torch tensor on the rank's GPU) is all-reduced
(sum) before the identical update on every rank - parameters stay in sync
without broadcasting.  Holdout evaluation is replicated (it is small).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .errors import PipelineError
from .featurizer import FEATURE_WIDTH, fit_normalizer, featurize_states, normalize


def flat_params(params) -> np.ndarray:
    return np.concatenate([np.ravel(params.Wx), np.ravel(params.Wh), np.ravel(params.b),
                           np.ravel(params.w), [float(params.b_out)]]).astype(np.float64)


def unflat_into(params, flat: np.ndarray):
    H = params.hidden
    G = 4 * H
    o = 0
    params.Wx = flat[o:o + 16 * G].reshape(16, G).copy(); o += 16 * G
    params.Wh = flat[o:o + H * G].reshape(H, G).copy(); o += H * G
    params.b = flat[o:o + G].copy(); o += G
    params.w = flat[o:o + H].copy(); o += H
    params.b_out = float(flat[o])
    return params


TRAIN_MODES = {"exact": 0, "tc": 1, "tcf": 2}  # TS_TRAIN_EXACT, TS_TRAIN_TC, TS_TRAIN_TCF


def shard(batch: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Contiguous shard of a global minibatch (sizes differ by at most one)."""
    n = len(batch)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return batch[lo:hi]


class DeviceGradients:
    """ts_train_* wrapper: dataset resident on the device.

    Host form: per-sample normalized matrices (full depth).  Device form
    (`from_device`): shared scheduled rows + prefix depths (bench)."""

    def __init__(self, ctx, X, Tlen, logt, hidden, mode="exact"):
        self.ctx = ctx
        self.hidden = hidden
        self.mode = mode
        self.n_params = 16 * 4 * hidden + hidden * 4 * hidden + 4 * hidden + hidden + 1
        if X is None:
            return
        X = np.ascontiguousarray(X, dtype=np.float64)
        T = np.ascontiguousarray(Tlen, dtype=np.int32)
        # sample i: rows[base_i + j] = its row of decision j = X[i, T_i - 1 - j]
        base = np.zeros(len(T), dtype=np.int64)
        np.cumsum(T[:-1], out=base[1:])
        rows = np.concatenate([X[i, : T[i]][::-1] for i in range(len(T))])
        rows = np.ascontiguousarray(rows)
        zeros = np.zeros(len(T), dtype=np.int32)
        depth = T.copy()  # every row scheduled
        logt = np.ascontiguousarray(logt, dtype=np.float64)
        ctx.check(ctx.lib.ts_train_load(
            ctx.h, _lib._p(rows), rows.shape[0], None, 0, _lib._p(base), _lib._p(zeros),
            _lib._p(T), _lib._p(depth), _lib._p(logt), len(T), hidden, 0))
        self.set_mode(mode)

    def set_mode(self, mode):
        if mode not in TRAIN_MODES:
            raise ValueError(f"training mode {mode!r} (expected one of {sorted(TRAIN_MODES)})")
        self.mode = mode
        self.ctx.check(self.ctx.lib.ts_train_set_mode(self.ctx.h, TRAIN_MODES[mode]))

    @classmethod
    def from_device(cls, ctx, d_rows, n_rows, d_init, n_init, d_row_base, d_init_base, d_T, d_depth,
                    d_logt, N, hidden, mode="exact"):
        self = cls(ctx, None, None, None, hidden)
        c = ctypes.c_void_p
        ctx.check(ctx.lib.ts_train_load(ctx.h, c(d_rows), n_rows, c(d_init), n_init, c(d_row_base),
                                        c(d_init_base), c(d_T), c(d_depth), c(d_logt), N, hidden, 1))
        self.set_mode(mode)
        return self

    def set_params(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        self.ctx.check(self.ctx.lib.ts_train_set_params(self.ctx.h, _lib._p(flat), flat.size))

    def get_params(self):
        out = np.empty(self.n_params)
        self.ctx.check(self.ctx.lib.ts_train_get_params(self.ctx.h, _lib._p(out), out.size))
        return out

    def grads(self, idx, n_total, target_scale, d_grad_ptr=None, raw_out=None):
        """raw_out: optional f64[len(idx)] host array receiving the forward raw."""
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        self.ctx.check(self.ctx.lib.ts_train_grads(
            self.ctx.h, _lib._p(idx), len(idx), int(n_total), float(target_scale),
            ctypes.c_void_p(d_grad_ptr) if d_grad_ptr else None,
            _lib._p(raw_out) if raw_out is not None else None))

    def apply(self, lr, clip, d_grad_ptr=None):
        self.ctx.check(self.ctx.lib.ts_train_apply(
            self.ctx.h, ctypes.c_void_p(d_grad_ptr) if d_grad_ptr else None, float(lr),
            float(clip), None))

    def forward(self, idx):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = np.empty(len(idx))
        self.ctx.check(self.ctx.lib.ts_train_forward(self.ctx.h, _lib._p(idx), len(idx),
                                                     _lib._p(out)))
        return out

    def sync(self):
        self.ctx.check(self.ctx.lib.ts_sync(self.ctx.h))


def _eval_split(dev, idxs, Tlen, logt_all, target_scale):
    """(mse, r2, median relative error) like value_model._eval_split: groups
    by sequence length in ascending order, entry order within a group."""
    idxs = np.asarray(idxs)
    order = idxs[np.argsort(Tlen[idxs], kind="stable")]
    raw = dev.forward(order)
    logt = logt_all[order]
    pred_log = raw + target_scale
    err = pred_log - logt
    mse = float(np.mean(err ** 2))
    ss_tot = float(np.sum((logt - logt.mean()) ** 2))
    r2 = 1.0 - float(np.sum(err ** 2)) / ss_tot if ss_tot > 0 else float(mse == 0.0)
    rel = np.abs(np.exp(pred_log) - np.exp(logt)) / np.exp(logt)
    return mse, r2, float(np.median(rel))


def train(params, dataset, cfg, device=None, dist=None, return_trace=False, mode="exact"):
    """Device-trained copy of `params` and the reference's metrics dict."""
    if len(dataset) < 10:
        raise PipelineError(f"dataset too small ({len(dataset)} < 10 entries)")
    targets = np.array([t for _, t in dataset], dtype=np.float64)
    if np.any(targets <= 0):
        bad = targets[targets <= 0][0]
        raise PipelineError(f"non-positive training target {bad}")
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    perm = rng.permutation(len(dataset))
    n_hold = max(1, int(round(len(dataset) * cfg.holdout_fraction)))
    hold, tr = perm[:n_hold], perm[n_hold:]

    mats = featurize_states([s for s, _ in dataset], device=device)
    params = params.copy()
    params.normalizer = fit_normalizer([mats[i] for i in tr])
    params.target_scale = float(np.mean(np.log(targets[tr])))

    Tlen = np.array([m.shape[0] for m in mats], dtype=np.int32)
    Tmax = int(Tlen.max())
    X = np.zeros((len(mats), Tmax, FEATURE_WIDTH))
    for i, m in enumerate(mats):
        X[i, : m.shape[0]] = normalize(params.normalizer, m)
    logt = np.log(targets)

    ctx = _lib.context(device)
    dev = DeviceGradients(ctx, X, Tlen, logt, params.hidden, mode=mode)
    dev.set_params(flat_params(params))

    rank, world, gbuf = 0, 1, None
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        import torch
        rank, world = dist.get_rank(), dist.get_world_size()
        gbuf = torch.zeros(dev.n_params, dtype=torch.float64, device=f"cuda:{ctx.device}")

    def step(batch):
        batch = batch[np.argsort(Tlen[batch], kind="stable")]  # _grouped: ascending length
        if gbuf is None:
            dev.grads(batch, len(batch), params.target_scale)
            dev.apply(lr, cfg.clip_norm)
            return
        import torch
        dev.grads(shard(batch, rank, world), len(batch), params.target_scale, gbuf.data_ptr())
        dev.sync()
        dist.all_reduce(gbuf)
        torch.cuda.synchronize(gbuf.device)
        dev.apply(lr, cfg.clip_norm, gbuf.data_ptr())

    best = dev.get_params()
    best_hold = _eval_split(dev, hold, Tlen, logt, params.target_scale)[0]
    stale = 0
    lr = cfg.learning_rate
    trace = []
    for _ in range(cfg.epochs):
        order = rng.permutation(len(tr))
        for start in range(0, len(tr), cfg.batch_size):
            step(tr[order[start:start + cfg.batch_size]])
        hold_mse = _eval_split(dev, hold, Tlen, logt, params.target_scale)[0]
        trace.append(hold_mse)
        if hold_mse < best_hold:
            best_hold = hold_mse
            best = dev.get_params()
            stale = 0
        else:
            stale += 1
            if stale % (cfg.patience // 2 or 1) == 0:
                lr *= 0.5
                dev.set_params(best)
            if stale >= cfg.patience:
                break
    dev.set_params(best)
    train_mse = _eval_split(dev, tr, Tlen, logt, params.target_scale)[0]
    hold_mse, r2, med = _eval_split(dev, hold, Tlen, logt, params.target_scale)
    unflat_into(params, best)
    metrics = {"train_mse": train_mse, "holdout_mse": hold_mse, "holdout_r2": r2,
               "holdout_median_rel_err": med}
    if return_trace:
        return params, metrics, trace
    return params, metrics


def gradients_samples_per_s(dev, idx_all, batch, target_scale, steps=20):
    """Throughput helper for bench: samples/s of device gradients."""
    import time
    dev.sync()
    t0 = time.perf_counter()
    n = 0
    for k in range(steps):
        b = idx_all[(k * batch) % len(idx_all):][:batch]
        dev.grads(b, len(b), target_scale)
        n += len(b)
    dev.sync()
    return n / (time.perf_counter() - t0)
