"""Cost oracle on the device against the reference's benchmark() on random
complete schedules (tests/golden/costs.json, two machine models), and the
device schedule generator against search.random_schedule."""

import ctypes
import json

import numpy as np
import pytest

from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss
from paper_2011_14486_b200.cost_oracle import MachineModel, cost_descriptor


@pytest.fixture(scope="module")
def costs(golden):
    return json.loads((golden / "costs.json").read_text())


def test_cost_descriptor_envelope(costs):
    for name, g in costs["pipelines"].items():
        p = pi.parse_pipeline(g["text"])
        d = cost_descriptor(p)
        assert d.size == len(p.stages) * (2 + 4 * 21)


@pytest.mark.gpu
def test_benchmark_matches_reference(costs):
    from paper_2011_14486_b200.cost_oracle import benchmark_states
    for mname, mw in costs["machines"].items():
        m = MachineModel(**mw)
        for name, g in costs["pipelines"].items():
            p = pi.parse_pipeline(g["text"])
            states = [ss.state_from_key(p, r["key"]) for r in g["states"]]
            got = benchmark_states(states, m)
            assert got == [int(r[mname]) for r in g["states"]], (mname, name)


@pytest.mark.gpu
def test_device_random_schedules_match_reference_walk(costs, gpu_ctx):
    import torch
    from paper_2011_14486_b200 import _lib
    for name in ("t5_diamond", "vgg16", "resnet18"):
        g = costs["pipelines"][name]
        p = pi.parse_pipeline(g["text"])
        inf = ss._info(p)
        pid = gpu_ctx.pipeline_id(inf.desc)
        n = len(g["states"])
        recs = torch.empty(n * inf.T * 16, dtype=torch.uint8, device="cuda")
        gpu_ctx.check(gpu_ctx.lib.ts_generate_schedules_device(gpu_ctx.h, pid, 1, 1, n, recs.data_ptr()))
        hr = np.frombuffer(recs.cpu().numpy().tobytes(), dtype=_lib.DECISION_DTYPE)
        for i in range(n):
            dec = [inf.decode(k, r).render() for k, r in enumerate(hr[i * inf.T:(i + 1) * inf.T])]
            assert p.name + "/" + ";".join(dec) == g["states"][i]["key"], (name, i)
