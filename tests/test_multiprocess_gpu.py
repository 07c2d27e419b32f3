"""The multi-process PRODUCT paths executed on the device: two ranks share
the one B200 (TS_DEVICE=0, gloo for the collectives - a correctness check of
the sharding, reduction and update logic with the device kernels in the loop,
not a scaling measurement).

* predict_states_sharded with the device scorer == single-process V, bit
  for bit (scoring has no data-path collective: each rank scores its slice).
* trainer.train(dist=...) (value_model.train semantics, value_model.py:
  241-293, under data parallelism: shard of every length-sorted minibatch,
  d_raw over the global size, all-reduced gradient, identical update) ==
  the single-process device trajectory.
* bench.py under torch.distributed.run with WORLD_SIZE=2 prints its line.
"""

import json
import os
import pathlib
import socket
import subprocess
import sys

import numpy as np
import pytest

from helpers import bits, pipeline_from, product_states

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, case):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TS_DEVICE="0")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_14486_b200.value_model import load
        params = load(ROOT / "tests" / "golden" / "v0.ckpt")
        if case == "score":
            from helpers import pipeline_from as pf, product_states as ps
            from paper_2011_14486_b200.distributed import predict_states_sharded
            z = dict(np.load(ROOT / "tests" / "golden" / "states_vgg16.npz"))
            states = ps(pf(z), z["keys"]) * 3
            q.put((rank, predict_states_sharded(params, states, dist)))
        else:
            from test_train import _dataset
            from paper_2011_14486_b200.trainer import flat_params, train
            from paper_2011_14486_b200.value_model import TrainConfig, init_params
            g, data = _dataset(ROOT / "tests" / "golden")
            c = g["config"]
            cfg = TrainConfig(c["learning_rate"], c["epochs"], c["batch_size"], c["seed"], c["clip_norm"],
                              c["holdout_fraction"], c["patience"])
            trained, metrics = train(init_params(c["seed"], c["hidden"]), data, cfg, dist=dist)
            q.put((rank, (flat_params(trained), metrics)))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return res


def test_sharded_device_scoring_bitwise(v0_path, state_sets):
    from paper_2011_14486_b200.value_model import load, predict_states
    z = state_sets["vgg16"]
    states = product_states(pipeline_from(z), z["keys"]) * 3
    want = predict_states(load(v0_path), states)
    res = _run("score")
    for r in (0, 1):
        assert np.array_equal(bits(res[r]), bits(want)), r


def test_data_parallel_device_training_matches_single_process(golden):
    from test_train import _dataset
    from paper_2011_14486_b200.trainer import flat_params, train
    from paper_2011_14486_b200.value_model import TrainConfig, init_params
    g, data = _dataset(golden)
    c = g["config"]
    cfg = TrainConfig(c["learning_rate"], c["epochs"], c["batch_size"], c["seed"], c["clip_norm"],
                      c["holdout_fraction"], c["patience"])
    single, m1 = train(init_params(c["seed"], c["hidden"]), data, cfg)
    want = flat_params(single)
    res = _run("train")
    p0, m0 = res[0]
    assert np.array_equal(bits(res[1][0]), bits(p0))  # ranks stay in sync without a broadcast
    err = np.max(np.abs(p0 - want) / np.maximum(np.abs(want), 1e-3))
    print(f"DP(2 ranks) vs single-process training: max param deviation {err:.2e}, holdout R^2 "
          f"{m0['holdout_r2']:.9f} vs {m1['holdout_r2']:.9f}")
    # the two differ only in the summation order of each minibatch's gradient
    # (two partial sums + all-reduce against one reduction): rounding-level,
    # measured 3e-13 over the whole run
    assert err < 1e-12, err
    assert abs(m0["holdout_r2"] - m1["holdout_r2"]) < 1e-12


def test_bench_two_ranks_prints_a_line():
    env = dict(os.environ, TS_DEVICE="0", TS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--states", "200000", "--no-cpu", "--no-greedy",
           "--train-pairs", "200000", "--train-batch", "1024", "--big-states", "0"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([t for t in r.stdout.splitlines() if t.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["v_training"]["parallelism"] == "dp2" and line["v_training"]["value"] > 0
    print(f"bench, 2 ranks on one GPU (gloo): {line['value']:.3e} states/s, training "
          f"{line['v_training']['value']:.3e} samples/s")
