"""Generate tests/golden/* by running the UNMODIFIED reference (oracle/_ref,
built by oracle/build_ref.sh from /root/reference).  Run in the build
container only (the GPU box has no /root/reference); the fixtures are
committed.

  python tools/make_golden.py

Produces
  v0.ckpt                 `tensched train <train assets> --rounds 0 --seed 0` (value_model.save)
  greedy.json             greedy_schedule under v0 for every asset/net: schedule text, visited,
                          predicted V of the final state (search.py:90-112, cli.py:231-238)
  noisy.json              noisy greedy (eps 0.25, SearchRng seeds) with the final rng state
  states_<pipeline>.npz   random partial states (SearchRng(seed): d = randrange(T)+1, then uniform
                          candidate choices): canonical keys, raw features (featurize_state),
                          V (predict_states, Cython backend)
  lstm_forward.npz        backend.lstm_forward on seeded random inputs
  candidates.json         candidate_actions renderings along seeded walks
"""

from __future__ import annotations

import json
import pathlib
import shutil
import subprocess
import sys
import tempfile

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF))

from tensched import backend  # noqa: E402
from tensched.featurizer import featurize_state  # noqa: E402
from tensched.pipeline_ir import parse_pipeline  # noqa: E402
from tensched.schedule_space import apply, candidate_actions, canonical_key, initial_state  # noqa: E402
from tensched.search import NoiseConfig, SearchRng, greedy_schedule, model_value  # noqa: E402
from tensched.value_model import load, predict, predict_states  # noqa: E402

STATE_COUNTS = {"vgg16": 48, "resnet18": 24, "resnet50": 6, "mobilenet_v2": 6}


def pipeline_files():
    files = sorted((REF / "assets" / "pipelines").rglob("*.pl"))
    files += sorted((ROOT / "assets" / "pipelines" / "nets").glob("*.pl"))
    return files


def rel(f: pathlib.Path) -> str:
    f = f.resolve()
    if f.is_relative_to(ROOT / "assets"):
        return str(f.relative_to(ROOT))
    return "ref:" + str(f.relative_to(REF / "assets"))


def random_partial(p, seed):
    rng = SearchRng(seed)
    d = rng.randrange(len(p.stages)) + 1
    s = initial_state(p)
    for _ in range(d):
        c = candidate_actions(s)
        s = apply(s, c[rng.randrange(len(c))])
    return s


def main():
    assert backend.BACKEND == "cython", backend.BACKEND
    GOLD.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([sys.executable, "-m", "tensched.cli", "train",
                        str(REF / "assets" / "pipelines" / "train"), "--out", td,
                        "--rounds", "0", "--seed", "0"], check=True,
                       env={"PYTHONPATH": str(REF), "PATH": "/usr/bin:/bin"})
        shutil.copy(pathlib.Path(td) / "v0.ckpt", GOLD / "v0.ckpt")
    params = load(GOLD / "v0.ckpt")
    V = model_value(params)

    greedy, noisy, cands = {}, {}, {}
    for f in pipeline_files():
        p = parse_pipeline(f.read_text())
        key = rel(f)
        s, visited = greedy_schedule(p, V)
        greedy[key] = {"pipeline": p.name, "text": f.read_text(), "schedule": [d.render() for d in s.decisions],
                       "visited": visited, "predicted": predict(params, s).hex()}
        print("greedy", key, visited, flush=True)
        if len(p.stages) <= 12:
            for seed in (3, 11):
                rng = SearchRng(seed)
                s2, v2 = greedy_schedule(p, V, NoiseConfig(0.25), rng)
                noisy[f"{key}#{seed}"] = {"schedule": [d.render() for d in s2.decisions],
                                          "visited": v2, "rng_state": rng.state}
        # candidate renderings along a seeded walk
        rng = SearchRng(5)
        s = initial_state(p)
        walk = []
        while not s.is_complete and len(walk) < 40:
            c = candidate_actions(s)
            walk.append([a.render() for a in c])
            s = apply(s, c[rng.randrange(len(c))])
        cands[key] = walk
        # random partial states
        n = STATE_COUNTS.get(p.name, 40)
        states = [random_partial(p, seed) for seed in range(1, n + 1)]
        feats = np.stack([featurize_state(s) for s in states])
        vals = predict_states(params, states)
        np.savez_compressed(GOLD / f"states_{p.name}.npz",
                            keys=np.array([canonical_key(s) for s in states]),
                            features=feats, values=vals,
                            seeds=np.arange(1, n + 1, dtype=np.int64), source=np.array(key),
                            text=np.array(f.read_text()))
    (GOLD / "greedy.json").write_text(json.dumps(greedy, indent=1, sort_keys=True) + "\n")
    (GOLD / "noisy.json").write_text(json.dumps(noisy, indent=1, sort_keys=True) + "\n")
    (GOLD / "candidates.json").write_text(json.dumps(cands, sort_keys=True) + "\n")

    rs = np.random.Generator(np.random.PCG64(1234))
    X = rs.normal(0.0, 2.0, (64, 34, 16))
    X[rs.random(X.shape) < 0.3] = 0.0  # exercise the zero skip
    raw = backend.lstm_forward(np.ascontiguousarray(X), params.Wx, params.Wh, params.b, params.w,
                               params.b_out)
    np.savez_compressed(GOLD / "lstm_forward.npz", X=X, raw=raw)
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
