import pathlib, sys, time
sys.path.insert(0, "/root/repo")
from paper_2011_14486_b200.pipeline_ir import parse_pipeline
from paper_2011_14486_b200.schedule_space import initial_state
from paper_2011_14486_b200.search import beam_search_gpu
from paper_2011_14486_b200.value_model import load
params = load("/root/repo/tests/golden/v0.ckpt")
for net in ("vgg16", "resnet18"):
    p = parse_pipeline(pathlib.Path(f"/root/repo/assets/pipelines/nets/{net}.pl").read_text())
    beam_search_gpu(initial_state(p), params, 8)
    t0 = time.perf_counter(); beam_search_gpu(initial_state(p), params, 8); print(net, (time.perf_counter()-t0)*1e3, "ms")
