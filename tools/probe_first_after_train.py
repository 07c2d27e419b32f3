"""Why the first greedy call per network is slow after bench's training leg:
runs bench.main (no CPU legs) with greedy_schedule_gpu wrapped so every
first call per pipeline is profiled (cProfile, top entries to stderr) with
the native layer-loop trace on.  Run on the GPU box."""
import cProfile
import io
import os
import pathlib
import pstats
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ["TS_GREEDY_TRACE"] = "1"
import paper_2011_14486_b200.search as S  # noqa: E402

orig = S.greedy_schedule_gpu
seen = set()


def wrapped(p, params, *a, **k):
    if p.name in seen:
        return orig(p, params, *a, **k)
    seen.add(p.name)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    out = orig(p, params, *a, **k)
    pr.disable()
    dt = time.perf_counter() - t0
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(14)
    print(f"=== first greedy {p.name}: {dt * 1e3:.1f} ms\n{s.getvalue()}", file=sys.stderr)
    return out


S.greedy_schedule_gpu = wrapped
sys.argv = ["bench.py", "--no-cpu", "--no-ref-greedy", "--no-exact", "--big-states", "0", "--steps", "2"]
import runpy  # noqa: E402
runpy.run_path(str(ROOT / "bench.py"), run_name="__main__")
