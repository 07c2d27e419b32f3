"""Value iteration (Alg. 2) on the device against the reference
(tests/golden/learner.json from tools/make_golden_learner.py): bootstrap
table identical, one value_iteration_round's refined table identical
(rollouts, beam completions, stitched costs), retrained model's metrics
close, evaluate_round report identical."""

import json

import pytest

from paper_2011_14486_b200 import pipeline_ir as pi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold(golden):
    return json.loads((golden / "learner.json").read_text())


def test_bootstrap_table_matches_reference(gold):
    from paper_2011_14486_b200.cost_oracle import MachineModel
    from paper_2011_14486_b200.learner import bootstrap
    pipes = [pi.parse_pipeline(t) for t in gold["pipelines"].values()]
    table = bootstrap(pipes, 20, MachineModel(), 0)
    assert table.serialize() == gold["bootstrap_table"]


def test_value_iteration_round_matches_reference(gold, v0_path):
    from paper_2011_14486_b200.cost_oracle import MachineModel
    from paper_2011_14486_b200.learner import (RoundConfig, bootstrap, evaluate_round,
                                               value_iteration_round)
    from paper_2011_14486_b200.search import NoiseConfig
    from paper_2011_14486_b200.value_model import TrainConfig, load
    c = gold["config"]
    pipes = [pi.parse_pipeline(t) for t in gold["pipelines"].values()]
    m = MachineModel()
    table = bootstrap(pipes, 20, m, 0)
    cfg = RoundConfig(schedules_per_pipeline=c["schedules_per_pipeline"], beam_width=c["beam_width"],
                      noise=NoiseConfig(c["epsilon"]),
                      train=TrainConfig(learning_rate=c["lr"], epochs=c["epochs"],
                                        batch_size=c["batch_size"], seed=c["train_seed"],
                                        patience=c["patience"]),
                      seed=c["seed"], hidden=32, machine=m)
    new_table, v1, metrics = value_iteration_round(pipes, load(v0_path), table, cfg)
    assert new_table.serialize() == gold["round_table"]
    for k in ("train_mse", "holdout_mse", "holdout_r2"):
        assert abs(metrics[k] - gold["metrics"][k]) <= 1e-4 * max(1.0, abs(gold["metrics"][k])), k
    assert evaluate_round(pipes, v1, m, 2, None).to_csv(1) == gold["report"]
