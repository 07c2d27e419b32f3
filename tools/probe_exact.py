"""The exact fp64 leg on device-resident VGG-16 sweep states: time per call
and per-kernel times (featurize<double> / k_score_exact32).
  python tools/probe_exact.py [n_states]"""
import ctypes
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

M = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
ctx = _lib.context(0)
ctx.set_params(load(ROOT / "tests/golden/v0.ckpt"))
inf = _info(parse_pipeline((ROOT / "assets/pipelines/nets/vgg16.pl").read_text()))
pid = ctx.pipeline_id(inf.desc)
dev = torch.device("cuda", 0)
recs = torch.empty(M * inf.T * 16, dtype=torch.uint8, device=dev)
offs = torch.empty(M + 1, dtype=torch.int64, device=dev)
nrec = ctypes.c_int64()
ctx.check(ctx.lib.ts_generate_states_device(ctx.h, pid, 1, M, recs.data_ptr(), offs.data_ptr(), ctypes.byref(nrec)))
out = torch.empty(M, dtype=torch.float64, device=dev)


def step():
    ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, nrec.value,
                                             _lib.MODE_EXACT, out.data_ptr()))


for _ in range(2):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    step()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
_t = np.zeros(4)
_c = np.zeros(4, dtype=np.int64)
ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
ctx.lib.ts_set_timing(ctx.h, 1)
step()
torch.cuda.synchronize()
ctx.lib.ts_set_timing(ctx.h, 0)
ctx.lib.ts_kernel_times(ctx.h, _lib._p(_t), _lib._p(_c), 1)
print(f"exact leg, {M} states: {dt * 1e3:.2f} ms/call = {M / dt / 1e6:.2f} M states/s; "
      f"kernel ms (featurize, -, lstm-exact, other) {np.round(_t, 3)}")
print("checksum", float(out.double().sum().item()))
