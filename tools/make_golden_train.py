"""Golden training fixtures from the UNMODIFIED reference (oracle/_ref).

Reproduces `tensched train <train assets> --rounds 0 --seed 0` step by step
(cli.py:187-192): bootstrap(...) -> train_on_table -> v0.ckpt, and records
the dataset in insertion order (learner.py:214-216) plus the metrics, so the
GPU trainer can be held to the reference trajectory.

  python tools/make_golden_train.py   -> tests/golden/train_v0.json
"""

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(REF))

from tensched.cost_oracle import MachineModel  # noqa: E402
from tensched.learner import RoundConfig, bootstrap, round_train_config  # noqa: E402
from tensched.pipeline_ir import parse_pipeline  # noqa: E402
from tensched.schedule_space import canonical_key  # noqa: E402
from tensched.value_model import TrainConfig, init_params, train  # noqa: E402


def main():
    files = sorted((REF / "assets" / "pipelines" / "train").glob("*.pl"))
    pipes = [parse_pipeline(f.read_text()) for f in files]
    base = TrainConfig(learning_rate=5e-2, epochs=600, batch_size=16, seed=0, patience=60)
    cfg = RoundConfig(train=round_train_config(base, 0), seed=0, hidden=32)
    table = bootstrap(pipes, 200, MachineModel(), 0)
    dataset = [(e.state, e.millis / 1000.0) for e in table.entries.values() if e.state]
    params = init_params(cfg.train.seed, cfg.hidden)
    trained, metrics = train(params, dataset, cfg.train)
    out = {
        "pipelines": {p.name: f.read_text() for p, f in zip(pipes, files)},
        "keys": [canonical_key(s) for s, _ in dataset],
        "targets": [t.hex() for _, t in dataset],
        "config": {"learning_rate": cfg.train.learning_rate, "epochs": cfg.train.epochs,
                   "batch_size": cfg.train.batch_size, "seed": cfg.train.seed,
                   "clip_norm": cfg.train.clip_norm,
                   "holdout_fraction": cfg.train.holdout_fraction,
                   "patience": cfg.train.patience, "hidden": cfg.hidden},
        "metrics": metrics,
        "b_out": trained.b_out.hex(), "target_scale": trained.target_scale.hex(),
    }
    (ROOT / "tests" / "golden" / "train_v0.json").write_text(json.dumps(out) + "\n")
    print(len(dataset), metrics)


if __name__ == "__main__":
    main()
