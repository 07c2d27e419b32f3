"""Device-resident scoring from 16-byte records vs 16-bit action codes
(ts_score_states_device vs ts_score_states_coded_device) on the bench's
12.5M VGG-16 sweep states; checks the two agree bit for bit.
Run on the GPU box: python tools/probe_coded_device.py"""
import ctypes
import pathlib
import sys

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
n = nrec.value
codes = torch.empty(n, dtype=torch.int16, device=dev)
ctx.check(ctx.lib.ts_encode_codes_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, codes.data_ptr()))
stream = torch.cuda.ExternalStream(ctx.lib.ts_stream(ctx.h), device=dev)
outs = {}
for name in ("records", "codes"):
    out = torch.empty(M, dtype=torch.float64, device=dev)

    def step():
        if name == "records":
            ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, n,
                                                     _lib.MODE_FAST, out.data_ptr()))
        else:
            ctx.check(ctx.lib.ts_score_states_coded_device(ctx.h, pid, codes.data_ptr(), offs.data_ptr(), M, n,
                                                           _lib.MODE_FAST, out.data_ptr()))
    for _ in range(3):
        step()
    times = np.zeros(4)
    counts = np.zeros(4, dtype=np.int64)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    ctx.lib.ts_set_timing(ctx.h, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.lib.ts_set_timing(ctx.h, 0)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {M / ms / 1e3:.1f} M states/s, {ms:.2f} ms/step, featurize {times[0] / max(counts[0], 1):.3f} ms, "
          f"lstm {times[2] / max(counts[2], 1):.3f} ms")
    outs[name] = out.cpu().numpy()
assert np.array_equal(outs["records"].view(np.uint64), outs["codes"].view(np.uint64))
print("bit-identical")
