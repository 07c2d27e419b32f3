"""Run the device gradients of one minibatch many times and check they are
bit-identical (mode exact / tc / tcf), plus the whole reference training
several times: a non-deterministic kernel shows up as differing bits."""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from test_train import _dataset  # noqa: E402
from paper_2011_14486_b200 import _lib  # noqa: E402
from paper_2011_14486_b200.featurizer import featurize_states, normalize  # noqa: E402
from paper_2011_14486_b200.trainer import DeviceGradients, flat_params, train  # noqa: E402
from paper_2011_14486_b200.value_model import TrainConfig, init_params, load  # noqa: E402

import torch  # noqa: E402

golden = ROOT / "tests" / "golden"
g, data = _dataset(golden)
params = load(golden / "v0.ckpt")
mats = featurize_states([s for s, _ in data])
T = np.array([m.shape[0] for m in mats], dtype=np.int32)
X = np.zeros((len(mats), T.max(), 16))
for i, m in enumerate(mats):
    X[i, : len(m)] = normalize(params.normalizer, m)
logt = np.log([t for _, t in data])
for mode in ("exact", "tc", "tcf"):
    dev = DeviceGradients(_lib.context(0), X, T, logt, params.hidden, mode=mode)
    dev.set_params(flat_params(params))
    rng = np.random.default_rng(5)
    bad = 0
    for trial in range(20):
        batch = rng.integers(0, len(mats), size=int(rng.integers(1, 64))).astype(np.int32)
        batch = batch[np.argsort(T[batch], kind="stable")]
        ref = None
        for rep in range(50):
            gb = torch.zeros(dev.n_params, dtype=torch.float64, device="cuda")
            dev.grads(batch, len(batch), params.target_scale, gb.data_ptr())
            dev.sync()
            v = gb.cpu().numpy().view(np.uint64).copy()
            if ref is None:
                ref = v
            elif not np.array_equal(v, ref):
                bad += 1
                print(mode, "trial", trial, "rep", rep, "B", len(batch), "differs in",
                      int(np.sum(v != ref)), "of", v.size)
                break
    print(mode, "gradient repeats differing:", bad)
c = g["config"]
cfg = TrainConfig(c["learning_rate"], c["epochs"], c["batch_size"], c["seed"], c["clip_norm"],
                  c["holdout_fraction"], c["patience"])
outs = []
for k in range(6):
    p, m = train(init_params(c["seed"], c["hidden"]), data, cfg)
    outs.append(flat_params(p).view(np.uint64).copy())
    print("train run", k, "holdout r2", m["holdout_r2"], "same as run 0:", np.array_equal(outs[-1], outs[0]))
