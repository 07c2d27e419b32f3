"""Where does the end-to-end (host-buffer) scoring time go?  Times
ts_score_states_packed on 2^20 VGG-16 sweep states for several chunk sizes
(TS_E2E_CHUNK), next to the bare H2D of the same bytes and the
device-resident call.  Run on the GPU box: python tools/probe_e2e.py"""
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

M = 1 << 20
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
n_records = nrec.value
out = torch.empty(M, dtype=torch.float64, device=dev)
stream = torch.cuda.ExternalStream(ctx.lib.ts_stream(ctx.h), device=dev)
h_recs = recs[: n_records * 16].cpu().numpy()
h_offs = offs.cpu().numpy()
packed = _lib.pack_records(np.frombuffer(h_recs.tobytes(), dtype=_lib.DECISION_DTYPE))
h_packed = torch.from_numpy(packed.view(np.int64)).pin_memory()
h_depth = torch.from_numpy(np.diff(h_offs).astype(np.uint8)).pin_memory()
h_out = torch.empty(M, dtype=torch.float64, pin_memory=True)
mode = _lib.MODE_FAST


def timed(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


def dev_step():
    ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, n_records, mode,
                                             out.data_ptr()))


d_buf = torch.empty(h_packed.numel(), dtype=torch.int64, device=dev)
print(f"device-resident step   {timed(dev_step):7.3f} ms")
_t = np.zeros(4)
_c = np.zeros(4, dtype=np.int64)
ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
ctx.lib.ts_set_timing(ctx.h, 1)
for _ in range(5):
    dev_step()
torch.cuda.synchronize()
ctx.lib.ts_set_timing(ctx.h, 0)
ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
print("  device-resident featurize/lstm/other ms", np.round(_t / 5, 3))
print(f"bare H2D {h_packed.numel() * 8 / 1e6:.0f} MB          {timed(lambda: d_buf.copy_(h_packed, non_blocking=True)):7.3f} ms")
from paper_2011_14486_b200.schedule_space import action_codes  # noqa: E402
codes = action_codes(inf, np.frombuffer(h_recs.tobytes(), dtype=_lib.DECISION_DTYPE), h_offs)
h_codes = torch.from_numpy(codes.view(np.int16)).pin_memory()
for chunk in (1 << 20, 1 << 19, 1 << 18, 1 << 17, 1 << 16):
    os.environ["TS_CODED_CHUNK"] = str(chunk)

    def coded():
        ctx.check(ctx.lib.ts_score_states_coded(ctx.h, pid, h_codes.data_ptr(), h_depth.data_ptr(), M, mode,
                                                h_out.data_ptr()))
    ms = timed(coded)
    times = np.zeros(4)
    counts = np.zeros(4, dtype=np.int64)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    ctx.lib.ts_set_timing(ctx.h, 1)
    for _ in range(5):
        coded()
    ctx.lib.ts_set_timing(ctx.h, 0)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    per = np.round(times / 5, 3)
    print(f"coded chunk {chunk:8d}   {ms:7.3f} ms  ({M / ms / 1e3:.1f} M states/s)  "
          f"featurize {per[0]} lstm {per[2]} other {per[3]} ms/call")
for chunk in (1 << 20, 1 << 18):
    os.environ["TS_E2E_CHUNK"] = str(chunk)

    def e2e():
        ctx.check(ctx.lib.ts_score_states_packed(ctx.h, pid, h_packed.data_ptr(), h_depth.data_ptr(), M, mode,
                                                 h_out.data_ptr()))
    ms = timed(e2e)
    print(f"e2e chunk {chunk:8d}     {ms:7.3f} ms  ({M / ms / 1e3:.1f} M states/s)")
