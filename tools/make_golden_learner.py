"""Golden value-iteration fixtures from the UNMODIFIED reference
(oracle/_ref): a small bootstrap table and one value_iteration_round
(learner.py:99-117, :221-249) + evaluate_round on the train assets.

  python tools/make_golden_learner.py -> tests/golden/learner.json
"""

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(REF))

from tensched.cost_oracle import MachineModel  # noqa: E402
from tensched.learner import RoundConfig, bootstrap, evaluate_round, value_iteration_round  # noqa: E402
from tensched.pipeline_ir import parse_pipeline  # noqa: E402
from tensched.search import NoiseConfig  # noqa: E402
from tensched.value_model import TrainConfig, load, predict  # noqa: E402


def main():
    files = sorted((REF / "assets" / "pipelines" / "train").glob("*.pl"))
    pipes = [parse_pipeline(f.read_text()) for f in files]
    m = MachineModel()
    table = bootstrap(pipes, 20, m, 0)
    v0 = load(ROOT / "tests" / "golden" / "v0.ckpt")
    cfg = RoundConfig(schedules_per_pipeline=2, beam_width=2, noise=NoiseConfig(0.25),
                      train=TrainConfig(learning_rate=5e-2, epochs=40, batch_size=16, seed=1,
                                        patience=60), seed=7920, hidden=32, machine=m)
    new_table, v1, metrics = value_iteration_round(pipes, v0, table, cfg)
    report = evaluate_round(pipes, v1, m, 2, None)
    out = {"pipelines": {p.name: f.read_text() for p, f in zip(pipes, files)},
           "bootstrap_table": table.serialize(), "round_table": new_table.serialize(),
           "metrics": metrics, "report": report.to_csv(1),
           "config": {"schedules_per_pipeline": 2, "beam_width": 2, "epsilon": 0.25,
                      "lr": 5e-2, "epochs": 40, "batch_size": 16, "train_seed": 1,
                      "patience": 60, "seed": 7920}}
    (ROOT / "tests" / "golden" / "learner.json").write_text(json.dumps(out) + "\n")
    print(len(table.entries), len(new_table.entries), metrics)
    print(report.to_csv(1))


if __name__ == "__main__":
    main()
