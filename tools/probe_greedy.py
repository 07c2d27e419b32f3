"""Greedy wall time on the benchmark networks (fused ts_greedy), repeated,
with the candidates visited and the distinct children rows (ts_greedy_stats)."""
import ctypes
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2011_14486_b200 import _lib  # noqa: E402
from paper_2011_14486_b200.pipeline_ir import parse_pipeline  # noqa: E402
from paper_2011_14486_b200.search import greedy_schedule_gpu  # noqa: E402
from paper_2011_14486_b200.value_model import load  # noqa: E402

params = load(ROOT / "tests/golden/v0.ckpt")
nets = sys.argv[1:] or ["resnet18", "resnet50", "mobilenet_v2"]
for net in nets:
    p = parse_pipeline((ROOT / f"assets/pipelines/nets/{net}.pl").read_text())
    greedy_schedule_gpu(p, params)
    t0 = time.perf_counter()
    for _ in range(3):
        s, visited = greedy_schedule_gpu(p, params)
    dt = (time.perf_counter() - t0) / 3
    ctx = _lib.context(0)
    vis, distinct = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.ts_greedy_stats(ctx.h, ctypes.byref(vis), ctypes.byref(distinct)))
    print(f"{net:14s} {dt * 1e3:7.1f} ms  visited {visited}  distinct rows {distinct.value}  "
          f"dedup {vis.value / max(distinct.value, 1):.3f}")
