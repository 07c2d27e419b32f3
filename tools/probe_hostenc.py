"""Host-encoder rates on the reference's own ScheduleState objects (VGG-16):
fresh walk states (new decision objects), clones (new objects, known
values), search-shaped children (shared decision objects), repeats."""
import gc
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
sys.path.insert(0, str(ROOT))
from tensched.pipeline_ir import parse_pipeline  # noqa: E402
from tensched.schedule_space import LayerSchedule, ScheduleState, apply, candidate_actions, initial_state  # noqa: E402
from tensched.search import SearchRng  # noqa: E402

import paper_2011_14486_b200.schedule_space as ss  # noqa: E402

p = parse_pipeline((ROOT / "assets" / "pipelines" / "nets" / "vgg16.pl").read_text())


def walkset(seed0, n):
    out = []
    for seed in range(seed0, seed0 + n):
        rng = SearchRng(seed)
        d = rng.randrange(len(p.stages)) + 1
        s = initial_state(p)
        for _ in range(d):
            c = candidate_actions(s)
            s = apply(s, c[rng.randrange(len(c))])
        out.append(s)
    return out


def clone(s):
    return ScheduleState(s.pipeline, tuple(LayerSchedule(d.stage, d.splits, d.order, d.vectorize_width, d.parallel,
                                                         d.compute_at, d.store_at) for d in s.decisions))


def rate(states):
    gc.disable()
    t0 = time.perf_counter()
    ss.encode_states(states)
    dt = time.perf_counter() - t0
    gc.enable()
    return len(states) / dt


ss.encode_states(walkset(99, 3))
for rep in range(3):
    print(f"fresh walk states: {rate(walkset(1 + 1000 * rep, 1000)):.0f} states/s")
base = walkset(50000, 1000)
ss.encode_states(base)
print(f"clones (new objects, seen values): {rate([clone(s) for s in base]):.0f} states/s")
kids = []
s = initial_state(p)
rng = SearchRng(7)
while not s.is_complete:
    c = candidate_actions(s)
    kids.extend(apply(s, a) for a in c)
    s = apply(s, c[rng.randrange(len(c))])
print(f"search children ({len(kids)}): {rate(kids):.0f} states/s")
print(f"repeat: {rate(kids):.0f} states/s")
