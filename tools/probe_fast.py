"""Quick probe of the FAST (tensor-core) path vs the exact path on golden states."""
import sys, pathlib, time
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests")); sys.path.insert(0, str(ROOT / "oracle"))
from helpers import pipeline_from, product_states
from paper_2011_14486_b200.value_model import load, predict_states, MODE_FAST, MODE_EXACT
v0 = load(ROOT / "tests/golden/v0.ckpt")
for f in sorted((ROOT / "tests/golden").glob("states_*.npz")):
    z = dict(np.load(f))
    p = pipeline_from(z)
    st = product_states(p, z["keys"])
    fast = predict_states(v0, st, mode=MODE_FAST)
    rel = np.abs(fast / z["values"] - 1)
    print(f"{p.name:16s} n={len(st):3d} max_rel={rel.max():.3e} mean_rel={rel.mean():.3e}", flush=True)
