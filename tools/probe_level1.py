"""Where the INTEGRATION level-1 V call spends its time on the reference's
own ScheduleState children of a VGG-16 walk: host encoding (cold) vs the
device call with records cached (first and repeat)."""
import sys, time
sys.path.insert(0, "."); sys.argv = ["x"]
import bench
bench._ref_import()
from tensched.pipeline_ir import parse_pipeline
from tensched.schedule_space import apply, candidate_actions, initial_state
from tensched.search import SearchRng
from tensched.value_model import load as ref_load
from paper_2011_14486_b200.search import model_value
import paper_2011_14486_b200.schedule_space as ss
params = ref_load("tests/golden/v0.ckpt")
p = parse_pipeline(bench.VGG.read_text())
def kids():
    rng = SearchRng(77); s = initial_state(p); out = []
    while not s.is_complete:
        c = candidate_actions(s); out.extend(apply(s, a) for a in c); s = apply(s, c[rng.randrange(len(c))])
    return out
V = model_value(params)
V(kids()[:64])
k = kids()
t0 = time.perf_counter(); ss.encode_states(k); t1 = time.perf_counter()
v = V(k); t2 = time.perf_counter()
v = V(k); t3 = time.perf_counter()
print(f"{len(k)} kids: encode {1e3*(t1-t0):.2f} ms, V (records cached) {1e3*(t2-t1):.2f} ms, V again {1e3*(t3-t2):.2f} ms")
