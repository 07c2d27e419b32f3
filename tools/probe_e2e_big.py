"""The bench's e2e leg (12.5 M VGG-16 sweep states, 16-bit codes from pinned
host buffers through ts_score_states_coded) against the device-resident
call, for several chunk schedules (TS_CODED_CHUNK / TS_CODED_STEP /
TS_ONE_LANE).  Run on the GPU box: python tools/probe_e2e_big.py"""
import ctypes
import os
import pathlib
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2011_14486_b200 import _lib  # noqa: E402
from paper_2011_14486_b200.pipeline_ir import parse_pipeline  # noqa: E402
from paper_2011_14486_b200.schedule_space import _info  # noqa: E402
from paper_2011_14486_b200.value_model import load  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 12_500_000
ctx = _lib.context(0)
ctx.set_params(load(ROOT / "tests/golden/v0.ckpt"))
inf = _info(parse_pipeline((ROOT / "assets/pipelines/nets/vgg16.pl").read_text()))
pid = ctx.pipeline_id(inf.desc)
T = inf.T
dev = torch.device("cuda", 0)
recs = torch.empty(M * T * 16, dtype=torch.uint8, device=dev)
offs = torch.empty(M + 1, dtype=torch.int64, device=dev)
nrec = ctypes.c_int64()
ctx.check(ctx.lib.ts_generate_states_device(ctx.h, pid, 1, M, recs.data_ptr(), offs.data_ptr(), ctypes.byref(nrec)))
n_rec = nrec.value
d_codes = torch.empty(n_rec, dtype=torch.int16, device=dev)
ctx.check(ctx.lib.ts_encode_codes_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, d_codes.data_ptr()))
out = torch.empty(M, dtype=torch.float64, device=dev)
h_codes = d_codes.cpu().pin_memory()
h_depth = torch.from_numpy(np.diff(offs.cpu().numpy()).astype(np.uint8)).pin_memory()
h_out = torch.empty(M, dtype=torch.float64, pin_memory=True)
mode = _lib.MODE_FAST


def timed(fn, k=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3, np.min(ts) * 1e3


def dev_step():
    ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, n_rec, mode,
                                             out.data_ptr()))


def dev_codes():
    ctx.check(ctx.lib.ts_score_states_coded_device(ctx.h, pid, d_codes.data_ptr(), offs.data_ptr(), M, n_rec,
                                                   mode, out.data_ptr()))


def coded():
    ctx.check(ctx.lib.ts_score_states_coded(ctx.h, pid, h_codes.data_ptr(), h_depth.data_ptr(), M, mode,
                                            h_out.data_ptr()))


print(f"M = {M}: device records {timed(dev_step)} ms, device codes {timed(dev_codes)} ms  (median, min)")
for env in ({}, {"TS_CODED_STEP": str(1 << 20)}, {"TS_CODED_CAP": str(1 << 22)},
            {"TS_CODED_CAP": str(1 << 22), "TS_CODED_CHUNK": str(1 << 17)}, {"TS_CODED_CAP": str(3 << 20)},
            {"TS_CODED_CHUNK": str(1 << 19)}):
    for k in ("TS_ONE_LANE", "TS_CODED_STEP", "TS_CODED_CHUNK", "TS_CODED_CAP"):
        os.environ.pop(k, None)
    os.environ.update(env)
    print(f"e2e coded {env or 'default'}: {timed(coded)} ms")

# kernel-time sums inside one e2e call (per-kernel CUDA events on each lane):
# if they add up to the device-resident call's, the gap is idle time
for k in ("TS_ONE_LANE", "TS_CODED_STEP", "TS_CODED_CHUNK"):
    os.environ.pop(k, None)
_t = np.zeros(4)
_c = np.zeros(4, dtype=np.int64)
for name, fn in (("device", dev_codes), ("e2e", coded)):
    fn()
    torch.cuda.synchronize()
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
    ctx.lib.ts_set_timing(ctx.h, 1)
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    ctx.lib.ts_set_timing(ctx.h, 0)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
    print(f"{name}: wall {wall:.2f} ms, featurize/lstm/other/... ms {np.round(_t, 3)} counts {_c}")
