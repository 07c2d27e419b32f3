"""First-call cost of the fused greedy per network, in a fresh process each:
host pipeline info (descriptor) vs the first ts_greedy vs a repeat."""
import pathlib
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, str(ROOT))
    net = sys.argv[2]
    from paper_2011_14486_b200 import _lib
    from paper_2011_14486_b200.pipeline_ir import parse_pipeline
    from paper_2011_14486_b200.schedule_space import _info
    from paper_2011_14486_b200.search import greedy_schedule_gpu
    from paper_2011_14486_b200.value_model import load
    params = load(ROOT / "tests/golden/v0.ckpt")
    _lib.context(0)
    warm = parse_pipeline((ROOT / "assets/pipelines/nets/crp2d.pl").read_text())
    greedy_schedule_gpu(warm, params)  # context, params upload, kernels loaded
    text = (ROOT / f"assets/pipelines/nets/{net}.pl").read_text()
    t0 = time.perf_counter()
    p = parse_pipeline(text)
    t1 = time.perf_counter()
    _info(p)
    t2 = time.perf_counter()
    greedy_schedule_gpu(p, params)
    t3 = time.perf_counter()
    greedy_schedule_gpu(p, params)
    t4 = time.perf_counter()
    print(f"{net:14s} parse {1e3 * (t1 - t0):6.2f} ms  info {1e3 * (t2 - t1):6.2f} ms  "
          f"first greedy {1e3 * (t3 - t2):6.2f} ms  repeat {1e3 * (t4 - t3):6.2f} ms")
else:
    for net in sys.argv[1:] or ["vgg16", "resnet18", "resnet50", "mobilenet_v2"]:
        subprocess.run([sys.executable, __file__, "--one", net], check=True)
