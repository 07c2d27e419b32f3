"""Parity at the bench's full size (BASELINE.json configs[3]: the VGG-16
scoring sweep, 12.5 M random partial schedules on one GPU - the exact
workload bench.py times, seeds 1..M).  The oracle cannot score 12.5 M states
in seconds, so the full batch is checked through size-independent
properties, and a sample spread over the whole batch against the oracle:

* every V finite and positive, in both legs;
* FAST within 1e-4 relative of EXACT on every state (north_star's fp32
  tolerance; tests/test_fast_leg.py states it per network);
* the e2e wire path (host codes + depths, ts_score_states_coded, chunked over
  two lanes) equals the device-resident call bit for bit, both legs;
* 1,000 states sampled across the batch (first, last, strided): EXACT equals
  the oracle bit for bit.
"""

import ctypes
import pathlib

import numpy as np
import pytest

import oracle as O
from helpers import bits, oracle_params, pipeline_from
from paper_2011_14486_b200 import _lib
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.value_model import MODE_EXACT, MODE_FAST, load

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent
M = 12_500_000  # bench.py --states default (one GPU)
FAST_RTOL = 1e-4


def test_full_size_sweep_properties(gpu_ctx, v0_path):
    import torch
    v0 = load(v0_path)
    p = pipeline_from({"text": (ROOT / "assets/pipelines/nets/vgg16.pl").read_text()})
    inf = ss._info(p)
    with gpu_ctx.lock:
        gpu_ctx.set_params(v0)
        pid = gpu_ctx.pipeline_id(inf.desc)
        recs = torch.empty(M * inf.T * 16, dtype=torch.uint8, device="cuda")
        offs = torch.empty(M + 1, dtype=torch.int64, device="cuda")
        nrec = ctypes.c_int64()
        gpu_ctx.check(gpu_ctx.lib.ts_generate_states_device(gpu_ctx.h, pid, 1, M, recs.data_ptr(),
                                                            offs.data_ptr(), ctypes.byref(nrec)))
        n_rec = nrec.value
        d_codes = torch.empty(n_rec, dtype=torch.int16, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_encode_codes_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M,
                                                         d_codes.data_ptr()))
        out = {}
        for mode in (MODE_EXACT, MODE_FAST):
            o = torch.empty(M, dtype=torch.float64, device="cuda")
            gpu_ctx.check(gpu_ctx.lib.ts_score_states_device(gpu_ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M,
                                                             n_rec, mode, o.data_ptr()))
            out[mode] = o.cpu().numpy()
        h_offs = offs.cpu().numpy()
        codes = d_codes.cpu().numpy().view(np.uint16)
        del d_codes
        depths = np.diff(h_offs).astype(np.uint8)
        wire = {}
        for mode in (MODE_EXACT, MODE_FAST):
            b = np.empty(M)
            gpu_ctx.check(gpu_ctx.lib.ts_score_states_coded(gpu_ctx.h, pid, _lib._p(codes), _lib._p(depths), M,
                                                            mode, _lib._p(b)))
            wire[mode] = b
        # a sample across the batch (first, last, strided) for the oracle
        idx = np.unique(np.concatenate([[0, M - 1], np.linspace(0, M - 1, 998).astype(np.int64)]))
        rows = np.concatenate([np.arange(h_offs[i], h_offs[i + 1]) for i in idx])
        sample = recs.view(-1, 16)[torch.from_numpy(rows).cuda()].cpu().numpy()
        h_recs = np.frombuffer(sample.tobytes(), dtype=_lib.DECISION_DTYPE)
        del recs
    ex, fa = out[MODE_EXACT], out[MODE_FAST]
    assert depths.min() >= 1 and depths.max() == inf.T  # the sweep's depths: 1..T
    for v in (ex, fa):
        assert np.all(np.isfinite(v)) and np.all(v > 0)
    rel = np.abs(fa - ex) / np.abs(ex)
    print(f"\n12.5 M VGG-16 states: FAST vs EXACT max rel {rel.max():.3e}, mean {rel.mean():.3e}")
    assert rel.max() <= FAST_RTOL, rel.max()
    for mode in (MODE_EXACT, MODE_FAST):
        assert np.array_equal(bits(wire[mode]), bits(out[mode])), mode
    # the sample against the oracle, bit for bit
    so = np.concatenate([[0], np.cumsum(depths[idx].astype(np.int64))])
    decs = [[O.as_act(inf.decode(k, r)) for k, r in enumerate(h_recs[so[j]:so[j + 1]])] for j in range(len(idx))]
    want = O.values(oracle_params(v0_path), O.Pipe(p), decs)
    assert np.array_equal(bits(ex[idx]), bits(want))
