"""Benchmark: candidate schedules scored per second (BASELINE.json metric) on
the synthetic scoring sweep - random partial schedules over VGG-16 (T=34),
scored with the v0 value function - plus the fused greedy wall times.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--states M] [--mode fast|exact]

One process per GPU (torchrun for N>1, NCCL only for the barrier and the
max-over-ranks reduction of the timings - scoring shards with no data-path
collective).  A step scores M states per GPU (default 12.5M, so that the
8-GPU run is BASELINE configs[3]'s 1e8-state sweep); states are generated on
the device by the reference's own random walk (SearchRng per state, untimed)
and stay resident in HBM; records (~3.5 GB per GPU) exceed the 126 MB L2,
so no explicit flush is needed between steps.

`value`  = states scored per second over all ranks, device-resident inputs.
`e2e`    = the same through the C-ABI with HOST buffers in the wire format
           predict_states uses for large batches (16-bit action codes + u8
           depths, ts_score_states_coded): H2D of the codes/depths and D2H of
           V inside the timed region.
`cpu_baseline` = the unmodified reference (oracle/_ref, tensched with its
           Cython kernel) on this host: predict_states on fresh VGG-16 states,
           one process and a pool of all cores.
`--impl reference` times that reference alone (rank 0) on the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import pathlib
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GOLD = ROOT / "tests" / "golden"
VGG = ROOT / "assets" / "pipelines" / "nets" / "vgg16.pl"
FLOPS_PER_STEP = 12352  # 2*48*128 MMA + 64 readout flops per state-timestep
RECORD_BYTES = 16
ROW_BYTES = 128
TRAFFIC_SOURCE = ("constant: dram__bytes_read.sum + dram__bytes_write.sum per state from one ncu --set full "
                  "capture at 12.5M states (profiles/), scaled to this launch; not measured in this run")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--states", type=int, default=12_500_000,
                    help="states per GPU per step (default: 1e8 over 8 GPUs)")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--cpu-states", type=int, default=1500, help="reference states per process")
    ap.add_argument("--cpu-repeats", type=int, default=10,
                    help="scoring passes over fresh copies of the reference states (~8 s of timed CPU work)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-greedy", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-pairs", type=int, default=10_000_000, help="training pairs per GPU")
    ap.add_argument("--train-batch", type=int, default=0,
                    help="per-GPU minibatch; 0 = 128 x the SM count (one 128-sequence tensor-core tile "
                         "per SM: 18,944 on a B200)")
    ap.add_argument("--big-states", type=int, default=100_000_000,
                    help="single-GPU sweep point (configs[3]'s 1e8 states on one GPU; 0 = skip)")
    ap.add_argument("--no-ref-greedy", action="store_true",
                    help="skip timing the reference's greedy_schedule on this host")
    ap.add_argument("--no-exact", action="store_true", help="skip the fp64 leg's sweep rate")
    ap.add_argument("--device-format", default="records", choices=["records", "codes"],
                    help="device-resident input format of the timed sweep")
    return ap.parse_args()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled every 5 ms through NVML (the
    same counters `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*`
    reads) on a background thread while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        import threading
        self.rows = []
        self.stop_ev = threading.Event()
        self.thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(index).uuid)
            except Exception:
                pass
            self.h = None
            if uuid:
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hh = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hh)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        self.h = hh
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            self.stop_ev.wait(0.005)

    def stop(self):
        if self.thread is None:
            return None
        self.stop_ev.set()
        self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "NVML, 5 ms"}


# --------------------------------------------------------------- reference (CPU)
def _ref_import():
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "tensched").exists():
        raise RuntimeError("oracle/_ref is not built (run oracle/build_ref.sh here)")
    sys.path.insert(0, str(ref))
    import tensched  # noqa: F401
    from tensched import backend
    assert backend.BACKEND == "cython"
    return ref


def _ref_worker(args):
    """Generate n fresh states with the reference's own walk (untimed), then
    time the reference's predict_states on them (features not cached)."""
    seed0, n, ckpt = args[:3]
    repeats = args[3] if len(args) > 3 else 1
    _ref_import()
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import apply, candidate_actions, initial_state
    from tensched.search import SearchRng
    from tensched.value_model import load, predict_states
    params = load(ckpt)
    p = parse_pipeline(VGG.read_text())
    walks = []
    for seed in range(seed0, seed0 + n):
        rng = SearchRng(seed)
        d = rng.randrange(len(p.stages)) + 1
        s = initial_state(p)
        acts = []
        for _ in range(d):
            c = candidate_actions(s)
            acts.append(c[rng.randrange(len(c))])
            s = apply(s, acts[-1])
        walks.append(acts)
    # `repeats` passes, each over FRESH state objects rebuilt from the walks'
    # actions (untimed), so no pass reuses the features the reference caches
    # on a state (featurizer.py:72-73)
    dt = 0.0
    for _ in range(repeats):
        states = []
        for acts in walks:
            s = initial_state(p)
            for a in acts:
                s = apply(s, a)
            states.append(s)
        t0 = time.perf_counter()
        predict_states(params, states, jobs=1)
        dt += time.perf_counter() - t0
    return dt, n * repeats


def cpu_reference(per_proc: int, seed0: int = 1, single: bool = True, repeats: int = 1):
    """The reference's own predict_states on fresh VGG-16 sweep states: one
    process, then a pool of os.cpu_count() processes over disjoint shards."""
    import multiprocessing as mp
    _ref_import()
    ckpt = str(GOLD / "v0.ckpt")
    out = {}
    if single:
        dt, n = _ref_worker((seed0, per_proc, ckpt, repeats))
        out["single"], out["single_sample"] = n / dt, n
    cores = os.cpu_count() or 1
    shards = [(seed0 + i * per_proc, per_proc, ckpt, repeats) for i in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_ref_worker, shards)
    out["pool"] = sum(r[1] for r in res) / max(r[0] for r in res)
    out["pool_sample"] = per_proc * cores * repeats
    out["cores"] = cores
    return out


def _ref_cost_worker(args):
    """The reference's cost_oracle.benchmark on n fresh complete VGG-16
    schedules (walks untimed)."""
    seed0, n = args
    _ref_import()
    from tensched.cost_oracle import MachineModel, benchmark
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import apply, candidate_actions, initial_state
    from tensched.search import SearchRng
    p = parse_pipeline(VGG.read_text())
    states = []
    for seed in range(seed0, seed0 + n):
        rng = SearchRng(seed)
        s = initial_state(p)
        while not s.is_complete:
            c = candidate_actions(s)
            s = apply(s, c[rng.randrange(len(c))])
        states.append(s)
    m = MachineModel()
    t0 = time.perf_counter()
    for s in states:
        benchmark(s, m)
    return n / (time.perf_counter() - t0)


def net_path(net):
    """Benchmark networks (assets/pipelines/nets) and the reference's own
    3-layer chain t3_chain (configs[0]: its copy in oracle/_ref/assets)."""
    if net == "t3_chain":
        return ROOT / "oracle" / "_ref" / "assets" / "pipelines" / "toys" / "t3_chain.pl"
    return ROOT / "assets" / "pipelines" / "nets" / f"{net}.pl"


def _ref_search_worker(task):
    """The reference's own search with its model_value V-callable
    (cli.py:cmd_schedule's timed region, cli.py:226-232) on one benchmark
    network, v0.ckpt: greedy_schedule, or beam_search(initial_state, V, 8)
    for ("beam", net).  Wall time, visited count (greedy) and the schedule."""
    kind, net = task
    _ref_import()
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import initial_state
    from tensched.search import beam_search, greedy_schedule, model_value
    from tensched.value_model import load
    params = load(str(GOLD / "v0.ckpt"))
    p = parse_pipeline(net_path(net).read_text())
    V = model_value(params)
    t0 = time.perf_counter()
    if kind == "beam":
        s, visited = beam_search(initial_state(p), V, 8), None
    else:
        s, visited = greedy_schedule(p, V)
    wall = time.perf_counter() - t0
    return task, wall, visited, [d.render() for d in s.decisions]


def reference_search(tasks):
    """One process per (kind, network) task (they run side by side on the
    host's cores; each wall time is its own process's)."""
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(len(tasks)) as pool:
        return {r[0]: r[1:] for r in pool.map(_ref_search_worker, tasks)}


def reference_gradients_rate(n=512, reps=3):
    """The reference's value_model.gradients (value_model.py:182-210, numpy
    BPTT) on n VGG-16 (partial schedule, target) pairs with their features
    cached ('samples/s, features cached'), this host,
    numpy's default BLAS threads."""
    _ref_import()
    from tensched.featurizer import featurize_state
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import apply, candidate_actions, initial_state
    from tensched.search import SearchRng
    from tensched.value_model import gradients, load
    params = load(str(GOLD / "v0.ckpt"))
    p = parse_pipeline(VGG.read_text())
    batch = []
    for seed in range(30_000_000, 30_000_000 + n):
        rng = SearchRng(seed)
        d = rng.randrange(len(p.stages)) + 1
        s = initial_state(p)
        for _ in range(d):
            c = candidate_actions(s)
            s = apply(s, c[rng.randrange(len(c))])
        featurize_state(s)  # cached on the state: timing covers the gradient only
        batch.append((s, 1000.0 + seed % 977))
    gradients(params, batch)
    t0 = time.perf_counter()
    for _ in range(reps):
        gradients(params, batch)
    return n * reps / (time.perf_counter() - t0)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    rates, ms = [], []
    per_proc = 800
    for step in range(args.warmup + args.steps):
        r = cpu_reference(per_proc, seed0=1 + step * 100003, single=False)
        if step >= args.warmup:
            rates.append(r["pool"])
            ms.append(r["pool_sample"] / r["pool"] * 1e3)  # scoring wall time of the step's sample
    v = sum(rates) / len(rates)
    line = {
        "metric": "candidate schedules scored/sec", "value": v, "unit": "states/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(ms) / len(ms), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "vgg16 synthetic scoring sweep (random partial schedules, "
                               "SearchRng walk, v0.ckpt)", "pipeline": "vgg16", "T": 34,
                   "states_per_step": per_proc * cores,
                   "note": "a bounded sample per step: the CPU reference takes ~1 h for 1e8 states"},
        "cpu_baseline": {"value": v, "unit": "states/s", "cores": cores, "kind": "reference",
                         "sample": "tensched.predict_states (Cython backend) on fresh VGG-16 "
                                   "states, a pool of os.cpu_count() processes per step"},
        "e2e": {"value": v, "unit": "states/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- V training
def train_throughput(ctx, pid, inf, params, rank, world, dev, args):
    """BASELINE configs[4]: V training on 10M (partial schedule, simulated
    cost) pairs over VGG-16, data parallel - the pairs are sharded across
    ranks (each rank holds 10M / world).  Per rank (untimed): complete random
    schedules on the device (search.random_schedule walk), their simulated
    costs from the device cost oracle (cost_oracle.benchmark), and every
    prefix of each schedule as a pair (learner.bootstrap without the
    cross-schedule min-aggregation), rows featurized once per schedule;
    65,536 pairs per rank are held out.  Timed: ONE EPOCH over the training
    pairs (a fresh permutation, global minibatch = per-rank batch x world) -
    gradients on the device, NCCL all-reduce of the 6,305-double gradient
    (N > 1), clip + SGD update - once per gradient mode.  Fit quality: the
    holdout MSE of log cost (value_model.loss) before and after the epoch."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2011_14486_b200 import _lib
    from paper_2011_14486_b200.cost_oracle import MachineModel, cost_descriptor
    from paper_2011_14486_b200.trainer import DeviceGradients, flat_params
    T = inf.T
    S_total = max(world, args.train_pairs // (T + 1))
    S = S_total // world
    seed0 = 10_000_000 + rank * S
    recs = torch.empty(S * T * 16, dtype=torch.uint8, device=dev)
    ctx.check(ctx.lib.ts_generate_schedules_device(ctx.h, pid, seed0, 1, S, recs.data_ptr()))
    offs = torch.arange(0, (S + 1) * T, T, dtype=torch.int64, device=dev)
    # simulated costs (device cost oracle; host-buffer API, untimed)
    h_recs = recs.cpu().numpy()
    h_offs = offs.cpu().numpy()
    cd = cost_descriptor(inf.p)
    limbs = np.empty((S, 4), dtype=np.uint64)
    mw = MachineModel().words()
    ctx.check(ctx.lib.ts_benchmark(ctx.h, pid, _lib._p(cd), cd.size, _lib._p(mw), _lib._p(h_recs),
                                   _lib._p(h_offs), S, _lib._p(limbs)))
    # the device cost oracle (cost_oracle.benchmark) through its
    # host-buffer C-ABI call, timed on a second pass (descriptor cached)
    t0 = time.perf_counter()
    ctx.check(ctx.lib.ts_benchmark(ctx.h, pid, _lib._p(cd), cd.size, _lib._p(mw), _lib._p(h_recs),
                                   _lib._p(h_offs), S, _lib._p(limbs)))
    cost_rate = S / (time.perf_counter() - t0)
    millis = [sum(int(limbs[i, k]) << (64 * k) for k in range(4)) for i in range(S)]
    logt_s = np.log(np.array([m / 1000.0 for m in millis]))
    rows = torch.empty((S * T, 16), dtype=torch.float64, device=dev)
    ctx.check(ctx.lib.ts_featurize_rows_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), S,
                                               rows.data_ptr()))
    init = torch.empty((T, 16), dtype=torch.float64, device=dev)
    ctx.check(ctx.lib.ts_init_rows(ctx.h, pid, 1, init.data_ptr()))
    N = S * (T + 1)
    sched = torch.arange(S, dtype=torch.int64, device=dev).repeat_interleave(T + 1)
    depth = torch.arange(T + 1, dtype=torch.int32, device=dev).repeat(S)
    row_base = sched * T
    init_base = torch.zeros(N, dtype=torch.int32, device=dev)
    Tl = torch.full((N,), T, dtype=torch.int32, device=dev)
    logt = torch.from_numpy(logt_s).to(dev)[sched]
    logt_h = logt.cpu().numpy()
    g = DeviceGradients.from_device(ctx, rows.data_ptr(), S * T, init.data_ptr(), T, row_base.data_ptr(),
                                    init_base.data_ptr(), Tl.data_ptr(), depth.data_ptr(),
                                    logt.data_ptr(), N, params.hidden)
    B = args.train_batch or 128 * torch.cuda.get_device_properties(dev).multi_processor_count
    rng = np.random.Generator(np.random.PCG64(1234 + rank))
    perm = rng.permutation(N).astype(np.int32)
    n_hold = min(65536, N // 10)
    hold, train_idx = perm[:n_hold], perm[n_hold:]
    # value_model.train's target scale: the mean log target of the training split
    tsum = torch.tensor([float(logt_h[train_idx].sum()), float(len(train_idx))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tsum)
    target_scale = float(tsum[0].item() / tsum[1].item())
    gbuf = torch.zeros(g.n_params, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(ctx.lib.ts_stream(ctx.h), device=dev)
    steps = len(train_idx) // B  # one epoch (every rank takes the same number of steps)
    if world > 1:
        st = torch.tensor([steps], dtype=torch.int64, device=dev)
        dist.all_reduce(st, op=dist.ReduceOp.MIN)
        steps = int(st.item())
    lr, clip = 1e-2, 5.0  # TrainConfig defaults (value_model.py:74-88)

    def holdout_mse():
        raw = np.concatenate([g.forward(hold[k:k + 16384]) for k in range(0, len(hold), 16384)])
        e = raw + target_scale - logt_h[hold]
        acc = torch.tensor([float(e @ e), float(len(e))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(acc)
        return float(acc[0].item() / acc[1].item())

    def epoch(order, n_steps):
        for k in range(n_steps):
            idx = order[k * B:(k + 1) * B]
            g.grads(idx, B * world, target_scale, gbuf.data_ptr())
            if world > 1:
                g.sync()
                dist.all_reduce(gbuf)
                torch.cuda.synchronize(dev)
            g.apply(lr, clip, gbuf.data_ptr())

    p0 = flat_params(params)

    def timed(mode):
        g.set_mode(mode)
        g.set_params(p0)
        before = holdout_mse()
        order = train_idx[rng.permutation(len(train_idx))]
        epoch(order, 3)  # warm-up steps, then back to p0
        g.set_params(p0)
        g.sync()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        epoch(order, steps)
        e1.record(stream)
        g.sync()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        assert np.all(np.isfinite(g.get_params()))
        after = holdout_mse()
        return float(ms.item()), before, after

    ms_exact, b_ex, a_ex = timed("exact")
    ms_tc, b_tc, a_tc = timed("tc")
    ms_tcf, b_tcf, a_tcf = timed("tcf")
    g.set_mode("exact")
    samples = B * world * steps
    # algorithmic weight-gradient flops of one step: 2 * 128 x 49 ([x | h_prev | 1])
    # per (sequence, timestep) pair; every sample of this dataset has T timesteps
    wg_flops = 2.0 * 128 * 49 * T * B
    # the model's dense contractions per (sequence, timestep): forward z
    # (2 x 48 x 128), BPTT dh (2 x 128 x 32), weight gradients (2 x 128 x 49)
    flops_st = 2.0 * (48 * 128 + 128 * 32 + 128 * 49)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak_tf = peaks.get("bf16_tflops", 1590.0)
    tf_tcf = flops_st * T * B * steps / (ms_tcf / 1e3) / 1e12
    return {"metric": "V-training samples/sec", "value": samples / (ms_tcf / 1e3),
            "mode": "tcf: forward AND BPTT recurrences on tcgen05 (split-fp16 UMMAs, fp32 TMEM "
                    "accumulation, MUFU gates; gradients within 1e-5 of fp64, tested)",
            "dtype": "f16x2 split operands (22-bit), f32 accumulation",
            "ms_per_step": ms_tcf / steps,
            "holdout_mse_log": {"before": b_tcf, "after_epoch": a_tcf},
            "tensor": {"algorithmic_tflops": tf_tcf, "peak": peak_tf, "frac": tf_tcf / peak_tf,
                       "algorithmic": "33,024 flops per sequence-timestep (forward z, BPTT dh, weight "
                                      "gradients); the split-fp16 UMMAs execute ~3x that"},
            "tc_weight_grads_only": {"value": samples / (ms_tc / 1e3), "ms_per_step": ms_tc / steps,
                                     "holdout_mse_log": {"before": b_tc, "after_epoch": a_tc},
                                     "mode": "tc: fp64 forward/BPTT, weight gradients on tcgen05 "
                                             "(3xTF32, TMEM, fused into BPTT)"},
            "cost_oracle": {"value": cost_rate, "unit": "complete VGG-16 schedules/s",
                            "note": "ts_benchmark (256-bit fixed point, exact), host buffers, per GPU"},
            "unit": "samples/s", "pairs_total": S * world * (T + 1), "pairs_per_gpu": N,
            "holdout_pairs_per_gpu": int(n_hold), "schedules_per_gpu": S, "batch_per_gpu": B,
            "global_batch": B * world, "steps": steps, "timed": "one epoch over the training pairs",
            "lr": lr, "clip_norm": clip,
            "weight_grad_tflops_per_step": wg_flops / 1e12,
            "exact": {"value": samples / (ms_exact / 1e3), "ms_per_step": ms_exact / steps,
                      "dtype": "f64", "holdout_mse_log": {"before": b_ex, "after_epoch": a_ex},
                      "note": "fp64 throughout: the reference's trajectory"},
            "parallelism": f"dp{world}", "collective": "NCCL all_reduce(sum) of the gradient"
                                                       if world > 1 else "none",
            "targets": "device cost oracle (cost_oracle.benchmark) of each prefix's schedule"}


# --------------------------------------------------------------- level 1: the V-callable
def v_callable_rate(params_path, seed=77):
    """INTEGRATION.md level 1: the reference's own ScheduleState objects scored
    through this package's V-callable (search.model_value, the seam of
    search.py:3-8).  The states are the reference's children along one VGG-16
    walk (apply(s, a) for every candidate of every layer: search-shaped, each
    child shares its parent's decision objects), built untimed by the
    reference; timed: V(children) - host encoding (csrc/hostenc.c) + device
    scoring + results - next to the reference's own model_value on the same
    objects (Cython, one process)."""
    _ref_import()
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import apply, candidate_actions, initial_state
    from tensched.search import SearchRng
    from tensched.search import model_value as ref_model_value
    from tensched.value_model import load as ref_load
    from paper_2011_14486_b200.search import model_value
    params = ref_load(str(params_path))
    p = parse_pipeline(VGG.read_text())

    def children_of_walk():
        rng = SearchRng(seed)
        s = initial_state(p)
        out = []
        while not s.is_complete:
            c = candidate_actions(s)
            out.extend(apply(s, a) for a in c)
            s = apply(s, c[rng.randrange(len(c))])
        return out
    V = model_value(params)
    V(children_of_walk()[:64])  # warm: pipeline descriptor, context
    kids = children_of_walk()
    t0 = time.perf_counter()
    v = V(kids)
    dt = time.perf_counter() - t0
    ref_kids = children_of_walk()
    t0 = time.perf_counter()
    rv = ref_model_value(params)(ref_kids)
    rdt = time.perf_counter() - t0
    import numpy as np
    same = bool(np.array_equal(np.asarray(v, dtype=np.float64).view(np.uint64),
                               np.asarray(rv, dtype=np.float64).view(np.uint64)))
    return {"states": len(kids), "value": len(kids) / dt, "unit": "states/s",
            "reference_1proc": len(ref_kids) / rdt, "bitwise_equal_to_reference": same,
            "note": "fresh reference ScheduleState children of one VGG-16 walk, V(children) through "
                    "search.model_value (exact leg) vs tensched.search.model_value (Cython)"}


# --------------------------------------------------------------- 1e8 states, one GPU
def big_sweep(ctx, pid, T, n_big, shard, mode, dev, stream, ref_out):
    """BASELINE configs[3]'s largest point on ONE GPU: n_big random partial
    VGG-16 schedules (seeds 1..n_big, the same walk as the main sweep),
    generated shard by shard on the device and kept as 16-bit action codes
    (2 B per decision).  `device`: scored device-resident, shard-sized calls
    over the one HBM-resident code array (absolute offsets).  `e2e`: the whole
    1e8 states in ONE ts_score_states_coded call from pinned host buffers
    (H2D of codes + depths and D2H of V inside the timed region)."""
    import numpy as np
    import torch
    from paper_2011_14486_b200 import _lib
    n_sh = -(-n_big // shard)
    recs = torch.empty(shard * T * 16, dtype=torch.uint8, device=dev)
    offs = torch.empty(shard + 1, dtype=torch.int64, device=dev)
    codes, depths = [], []
    t_gen = time.perf_counter()
    for k in range(n_sh):
        m = min(shard, n_big - k * shard)
        nrec = ctypes.c_int64()
        ctx.check(ctx.lib.ts_generate_states_device(ctx.h, pid, 1 + k * shard, m, recs.data_ptr(),
                                                    offs.data_ptr(), ctypes.byref(nrec)))
        c = torch.empty(max(nrec.value, 1), dtype=torch.int16, device=dev)
        ctx.check(ctx.lib.ts_encode_codes_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), m, c.data_ptr()))
        codes.append(c[: nrec.value])
        depths.append((offs[1: m + 1] - offs[:m]).to(torch.uint8))
    del recs, offs
    d_codes = torch.cat(codes)
    del codes
    d_depth = torch.cat(depths)
    del depths
    d_offs = torch.zeros(n_big + 1, dtype=torch.int64, device=dev)
    d_offs[1:] = torch.cumsum(d_depth.to(torch.int64), 0)
    n_rec = int(d_offs[-1].item())
    t_gen = time.perf_counter() - t_gen
    d_out = torch.empty(n_big, dtype=torch.float64, device=dev)
    bounds = [(k * shard, min(n_big, (k + 1) * shard)) for k in range(n_sh)]
    h_off = d_offs.cpu().numpy()

    def dev_step():
        for s0, s1 in bounds:
            r = int(h_off[s1] - h_off[s0]) if mode == _lib.MODE_FAST else n_rec
            ctx.check(ctx.lib.ts_score_states_coded_device(
                ctx.h, pid, d_codes.data_ptr(), d_offs.data_ptr() + 8 * s0, s1 - s0, r, mode,
                d_out.data_ptr() + 8 * s0))

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    ms_dev = timed(dev_step, 2)
    h_codes = torch.empty(n_rec, dtype=torch.int16, pin_memory=True)
    h_codes.copy_(d_codes)
    h_depth = torch.empty(n_big, dtype=torch.uint8, pin_memory=True)
    h_depth.copy_(d_depth)
    h_out = torch.empty(n_big, dtype=torch.float64, pin_memory=True)
    del d_codes, d_depth

    def e2e_step():
        ctx.check(ctx.lib.ts_score_states_coded(ctx.h, pid, h_codes.data_ptr(), h_depth.data_ptr(), n_big, mode,
                                                h_out.data_ptr()))
    ms_e2e = timed(e2e_step, 2)
    v_dev = d_out.cpu().numpy()
    assert np.array_equal(h_out.numpy(), v_dev), "1e8 point: e2e and device-resident V differ"
    m0 = min(len(ref_out), n_big)
    assert np.array_equal(v_dev[:m0], ref_out[:m0]), "1e8 point: first shard differs from the main sweep"
    assert np.all(np.isfinite(v_dev)) and np.all(v_dev > 0)
    return {"states": n_big, "records": n_rec, "value": n_big / (ms_dev / 1e3), "ms": ms_dev,
            "e2e": {"value": n_big / (ms_e2e / 1e3), "ms": ms_e2e, "h2d_bytes": 2 * n_rec + n_big,
                    "d2h_bytes": 8 * n_big, "call": "one ts_score_states_coded call, pinned host buffers"},
            "unit": "states/s", "generate_s": round(t_gen, 1),
            "note": f"{n_sh} shard-sized device-resident calls over one HBM-resident code array; the "
                    "first shard's V equals the main sweep's bit for bit"}


# --------------------------------------------------------------- GPU arm
def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one GPU per rank (LOCAL_RANK); TS_DEVICE / TS_DIST_BACKEND=gloo let the
    # multi-process test run two ranks on one GPU (correctness only)
    local = int(os.environ.get("TS_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("TS_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2011_14486_b200 import _lib
    from paper_2011_14486_b200.pipeline_ir import parse_pipeline
    from paper_2011_14486_b200.schedule_space import _info
    from paper_2011_14486_b200.value_model import load

    ctx = _lib.context(local)
    params = load(GOLD / "v0.ckpt")
    ctx.set_params(params)
    p = parse_pipeline(VGG.read_text())
    inf = _info(p)
    pid = ctx.pipeline_id(inf.desc)
    T = inf.T
    M = args.states
    mode = _lib.MODE_FAST if args.mode == "fast" else _lib.MODE_EXACT
    dev = torch.device("cuda", local)

    # ---- untimed: generate this rank's shard of states on the device
    seed0 = 1 + rank * M
    recs = torch.empty(M * T * 16, dtype=torch.uint8, device=dev)
    offs = torch.empty(M + 1, dtype=torch.int64, device=dev)
    nrec = ctypes.c_int64()
    ctx.check(ctx.lib.ts_generate_states_device(ctx.h, pid, seed0, M, recs.data_ptr(),
                                                offs.data_ptr(), ctypes.byref(nrec)))
    n_records = nrec.value
    out = torch.empty(M, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(ctx.lib.ts_stream(ctx.h), device=dev)

    # device-resident wire format: 16-bit action codes (2 B per decision,
    # decoded through the L2-resident code table) or the 16-byte records
    d_codes = torch.empty(max(n_records, 1), dtype=torch.int16, device=dev)
    ctx.check(ctx.lib.ts_encode_codes_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M, d_codes.data_ptr()))
    dev_fmt = args.device_format

    def step():
        if dev_fmt == "codes":
            ctx.check(ctx.lib.ts_score_states_coded_device(ctx.h, pid, d_codes.data_ptr(), offs.data_ptr(), M,
                                                           n_records if mode != _lib.MODE_FAST else n_records,
                                                           mode, out.data_ptr()))
        else:
            ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M,
                                                     n_records, mode, out.data_ptr()))

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    vals = out.cpu().numpy()
    assert np.all(np.isfinite(vals)) and np.all(vals > 0), "non-positive V"

    # ---- device-resident timed region
    times = np.zeros(4)
    counts = np.zeros(4, dtype=np.int64)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    ctx.lib.ts_set_timing(ctx.h, 1)
    launches0 = ctx.launches()
    clocks = ClockSampler(local)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ctx.lib.ts_set_timing(ctx.h, 0)
    ctx.lib.ts_kernel_times(ctx.h, _lib._p(times), _lib._p(counts), 1)
    launches = ctx.launches() - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_states = M * world * args.steps
    value = total_states / (ms_max / 1e3)

    # ---- e2e: host buffers through the C-ABI (pinned), H2D + D2H inside
    h_offs = torch.empty(M + 1, dtype=torch.int64, pin_memory=True)
    h_offs.copy_(offs)
    h_out = torch.empty(M, dtype=torch.float64, pin_memory=True)
    # the wire format predict_states sends for large batches: 16-bit action
    # codes (ts_score_states_coded), every decision of these walks being in
    # candidate_actions' space; prepared outside the timed region (encoded
    # on the device here, as schedule_space.action_codes does on the host)
    h_wire = torch.empty(n_records, dtype=torch.int16, pin_memory=True)
    h_wire.copy_(d_codes[:n_records])
    h_depth = torch.empty(M, dtype=torch.uint8, pin_memory=True)
    h_depth.copy_((offs[1:] - offs[:-1]).to(torch.uint8))
    wire_name = "16-bit action codes + u8 depths (ts_score_states_coded)"
    wire_fn = ctx.lib.ts_score_states_coded
    e2e_h2d = int(h_wire.numel() * h_wire.element_size() + M)

    def e2e_step():
        ctx.check(wire_fn(ctx.h, pid, h_wire.data_ptr(), h_depth.data_ptr(), M, mode, h_out.data_ptr()))

    for _ in range(2):
        e2e_step()
    barrier()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(args.steps):
        e2e_step()
    ev3.record(stream)
    barrier()
    t2 = torch.tensor([ev2.elapsed_time(ev3)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = total_states / (float(t2.item()) / 1e3)
    assert np.allclose(h_out.numpy(), out.cpu().numpy(), rtol=0, atol=0)

    # ---- the exact fp64 leg on the same states (device-resident; the
    # precision the reference computes in, what the greedy parity uses)
    exact_leg = None
    if mode == _lib.MODE_FAST and not args.no_exact:
        out_ex = torch.empty(M, dtype=torch.float64, device=dev)

        def ex_step():
            ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), M,
                                                     n_records, _lib.MODE_EXACT, out_ex.data_ptr()))
        ex_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(2):
            ex_step()
        e1.record(stream)
        barrier()
        tx = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tx, op=dist.ReduceOp.MAX)
        rel = (out / out_ex - 1).abs().max().item()
        exact_leg = {"value": 2 * M * world / (float(tx.item()) / 1e3), "unit": "states/s", "dtype": "f64",
                     "ms_per_step": float(tx.item()) / 2, "steps": 2,
                     "fast_vs_exact_max_rel": rel,
                     "note": "same states, device-resident; fp64 in the Cython kernel's operation order"}
        del out_ex

    # ---- roofline of the dominant kernel
    offs_h = h_offs.numpy()
    depths = np.diff(offs_h)
    timesteps = int(depths.sum())
    names = ["featurize", "lstm_exact", "lstm_fast", "other"]
    avg = {names[k]: times[k] / counts[k] for k in range(4) if counts[k]}
    dom = max(avg, key=lambda k: times[names.index(k)])
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    # ncu --set full captures (profiles/r02_ncu.md): DRAM bytes per state of each
    # kernel at 12.5M states (this bench's default launch), scaled to this launch
    traffic_per_state = {"featurize": (6.285197e9 + 7.072871e9) / 12.5e6,
                         "lstm_fast": (8.762989e9 + 0.379514e9) / 12.5e6}
    row_bytes = 32 if mode == _lib.MODE_FAST else ROW_BYTES  # FAST rows: 8 acquired f32
    if dom == "featurize":
        # SURVEY 8(d)'s per-unit figure: decision records read (32 B per
        # scheduled stage) + the state's feature matrix written (128 B per
        # row, all T rows); the kernel physically moves far less (16 B
        # records or 2 B codes, 32 B acquired rows for scheduled stages only:
        # `physical`), which is why it is issue-bound rather than HBM-bound
        bytes_per_launch = n_records * 32 + M * T * ROW_BYTES
        achieved = bytes_per_launch / (avg[dom] / 1e3) / 1e9
        phys = n_records * (RECORD_BYTES + row_bytes) + 8 * (M + 1)
        peak = peaks.get("hbm_gbs", 6650.0)
        tr = traffic_per_state.get(dom)
        roof = {"kernel": "k_featurize_rows", "bound": "hbm", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr * M if tr and mode == _lib.MODE_FAST else None,
                "traffic_source": TRAFFIC_SOURCE,
                "bytes_per_launch": bytes_per_launch,
                "algorithmic": "SURVEY 8(d): 32 B per scheduled stage (records) + 128 B x T (feature rows)",
                "physical": {"bytes_per_launch": phys, "achieved_gbs": phys / (avg[dom] / 1e3) / 1e9,
                             "what": f"16 B record read + {row_bytes} B row written per scheduled stage"}}
    else:
        # SURVEY 8(d)'s per-unit figure: 12,352 flops per state-timestep over
        # the full state (T timesteps); the kernel executes only the
        # scheduled timesteps (the shared unscheduled prefix is computed once
        # per pipeline): `executed`
        flops_per_launch = FLOPS_PER_STEP * T * M
        achieved = flops_per_launch / (avg[dom] / 1e3) / 1e12
        executed = FLOPS_PER_STEP * timesteps
        peak = peaks.get("bf16_tflops", 1590.0)
        tr = traffic_per_state.get(dom)
        roof = {"kernel": "k_lstm_tc" if dom == "lstm_fast" else "k_score_exact", "bound": "tensor",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": tr * M if tr else None, "traffic_source": TRAFFIC_SOURCE,
                "flops_per_launch": flops_per_launch,
                "algorithmic": "SURVEY 8(d): 12352 flops per state-timestep x T timesteps per state",
                "executed": {"flops_per_launch": executed,
                             "achieved_tflops": executed / (avg[dom] / 1e3) / 1e12,
                             "what": "scheduled timesteps only (shared unscheduled prefix computed once)"}}
    roof["kernel_ms"] = {k: round(v, 4) for k, v in avg.items()}
    if "lstm_fast" in avg:
        # the LSTM's binding unit: 5 ex2 + 1 rcp per hidden unit and
        # timestep (pairs of units share a reciprocal) = 192 MUFU ops per
        # state-timestep against 16 MUFU ops/clk/SM
        mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965
        mufu_peak = 16 * (torch.cuda.get_device_properties(dev).multi_processor_count) * mhz * 1e6
        mufu = 192.0 * timesteps / (avg["lstm_fast"] / 1e3)
        roof["k_lstm_tc_mufu"] = {"bound": "xu (MUFU)", "achieved": mufu / 1e12, "peak": mufu_peak / 1e12,
                                  "unit": "Tops/s", "frac": mufu / mufu_peak,
                                  "algorithmic": "192 MUFU ops per state-timestep (5 ex2 + 1 rcp per unit)"}
    if "featurize" in avg and mode == _lib.MODE_FAST:
        # the featurizer's binding resource is instruction issue (integer
        # walk): warp instructions per scheduled row from the ncu capture
        # (6.3449e9 warp instructions for 12.5M states = 218.7M rows,
        # profiles/r02_ncu.md), against 4 warp instructions / clk / SM
        mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965
        issue_peak = 4 * torch.cuda.get_device_properties(dev).multi_processor_count * mhz * 1e6
        issued = 6.344893e9 / 218.7e6 * timesteps / (avg["featurize"] / 1e3)
        roof["k_featurize_rows_issue"] = {"bound": "issue", "achieved": issued / 1e12, "peak": issue_peak / 1e12,
                                          "unit": "T warp-instr/s", "frac": issued / issue_peak,
                                          "algorithmic": "29.0 warp instructions per scheduled row (ncu)",
                                          "instructions_source": "constant from one ncu --set full "
                                                                 "capture (profiles/r02_ncu.md), not "
                                                                 "measured in this run"}
    roof["note"] = ("neither kernel is HBM- or tensor-bound: k_lstm_tc is MUFU/issue-bound (XU pipe 83%, "
                    "issue 61% in ncu; k_lstm_tc_mufu), k_featurize_rows is ALU/issue-bound integer work; "
                    "profiles/r02_ncu.md")

    # ---- batch-size sweep (1e4..1e7 states per GPU), device-resident,
    # on prefixes of this rank's states: where launch latency stops mattering
    sweep = {}
    for n_sw in (10 ** 4, 10 ** 5, 10 ** 6, 10 ** 7):
        if n_sw > M:
            break
        nr_sw = int(offs[n_sw].item())
        out_sw = out[:n_sw]

        def sw_step():
            ctx.check(ctx.lib.ts_score_states_device(ctx.h, pid, recs.data_ptr(), offs.data_ptr(), n_sw,
                                                     nr_sw, mode, out_sw.data_ptr()))
        sw_step()
        reps = max(3, min(50, int(2e7 // n_sw)))
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            sw_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        sweep[f"{n_sw:.0e}"] = round(n_sw * reps / (e0.elapsed_time(e1) / 1e3), 1)

    big = None
    if args.big_states and world == 1 and args.big_states > M:
        vals_main = out.cpu().numpy()
        big = big_sweep(ctx, pid, T, args.big_states, M, mode, dev, stream, vals_main)
        sweep[f"{args.big_states:.0e}"] = round(big["value"], 1)
        torch.cuda.empty_cache()

    train_line = None
    if not args.no_train:
        train_line = train_throughput(ctx, pid, inf, params, rank, world, dev, args)

    greedy, beam, level1 = {}, {}, None
    if rank == 0 and not args.no_greedy:
        from paper_2011_14486_b200.search import greedy_schedule_gpu
        for net in ("t3_chain", "crp2d", "vgg16", "resnet18", "resnet50", "mobilenet_v2"):
            if not net_path(net).exists():
                continue
            pn = parse_pipeline(net_path(net).read_text())
            t0 = time.perf_counter()
            greedy_schedule_gpu(pn, params)  # first call: descriptor upload, init rows, prefix states
            first = time.perf_counter() - t0
            t0 = time.perf_counter()
            s, visited = greedy_schedule_gpu(pn, params)
            wall = time.perf_counter() - t0
            vis, distinct = ctypes.c_int64(), ctypes.c_int64()
            ctx.check(ctx.lib.ts_greedy_stats(ctx.h, ctypes.byref(vis), ctypes.byref(distinct)))
            greedy[net] = {"wall_s": round(wall, 4), "first_call_s": round(first, 4), "visited": visited,
                           "candidates_per_s": round(visited / wall, 1),
                           "distinct_children": int(distinct.value),
                           "dedup_factor": round(visited / max(1, distinct.value), 3),
                           "schedule": [d.render() for d in s.decisions]}
        from paper_2011_14486_b200.schedule_space import initial_state
        from paper_2011_14486_b200.search import beam_search_gpu
        for net in ("vgg16", "resnet18"):  # beam_search(initial_state, model_value(v0), 8)
            pn = parse_pipeline((ROOT / "assets" / "pipelines" / "nets" / f"{net}.pl").read_text())
            t0 = time.perf_counter()
            beam_search_gpu(initial_state(pn), params, 8)
            first = time.perf_counter() - t0
            t0 = time.perf_counter()
            s = beam_search_gpu(initial_state(pn), params, 8)
            beam[net] = {"wall_s": round(time.perf_counter() - t0, 4), "first_call_s": round(first, 4),
                         "width": 8, "schedule": [d.render() for d in s.decisions]}
        try:  # in a fresh process, like a user's: this one holds the bench's
            # buffers and objects (its collector passes and allocator state
            # slowed the Python-side encoding ~4x)
            import multiprocessing as mp
            with mp.get_context("spawn").Pool(1) as pool:
                level1 = pool.apply(v_callable_rate, (GOLD / "v0.ckpt",))
            level1["process"] = "fresh (spawned) process, its own CUDA context"
        except Exception as e:  # reported, never silently replaced
            level1 = {"unavailable": str(e)}
        if not args.no_ref_greedy:
            try:
                tasks = [("greedy", n) for n in greedy] + [("beam", n) for n in beam]
                ref = reference_search(tasks)
                for (kind, net), (wall, visited, sched) in ref.items():
                    mine = greedy[net] if kind == "greedy" else beam[net]
                    mine["reference"] = {
                        "wall_s": round(wall, 3), "visited": visited,
                        "identical_schedule": sched == mine["schedule"] and (
                            kind == "beam" or visited == mine["visited"]),
                        "kind": f"tensched.search.{'greedy_schedule' if kind == 'greedy' else 'beam_search'}"
                                " + model_value (Cython), oracle/_ref, one process per task on this host"}
                    mine["speedup_vs_reference"] = round(wall / mine["wall_s"], 1)
            except Exception as e:  # reported, never silently replaced
                greedy["reference"] = f"unavailable: {e}"
        for g_ in list(greedy.values()) + list(beam.values()):
            if isinstance(g_, dict):
                g_.pop("schedule", None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline: rank 0 at N=1 only
        try:
            r = cpu_reference(args.cpu_states, repeats=args.cpu_repeats)
            cpu = {"value": r["pool"], "unit": "states/s", "cores": r["cores"], "kind": "reference",
                   "single_process": r["single"],
                   "sample": f"tensched predict_states (Cython) on fresh VGG-16 sweep states: "
                             f"{r['single_sample']} states in 1 process, {r['pool_sample']} over "
                             f"{r['cores']} processes ({args.cpu_states} walks per process, "
                             f"scored {args.cpu_repeats}x as fresh state objects, so features are "
                             f"recomputed every pass)"}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "states/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
        if train_line is not None and cpu is not None and cpu.get("value"):
            try:  # the reference's cost oracle, one process, next to the device one
                train_line["cost_oracle"]["cpu_reference_1proc"] = _ref_cost_worker((5_000_000, 100))
            except Exception as e:
                train_line["cost_oracle"]["cpu_reference_1proc"] = f"unavailable: {e}"
            try:  # the reference's own gradients (numpy BPTT), features cached
                train_line["cpu_reference"] = {
                    "value": reference_gradients_rate(), "unit": "samples/s",
                    "what": "tensched.value_model.gradients on 512 VGG-16 pairs (T=34), features cached, "
                            "numpy default BLAS threads, this host"}
            except Exception as e:
                train_line["cpu_reference"] = f"unavailable: {e}"

    if rank == 0:
        line = {
            "metric": "candidate schedules scored/sec", "value": value, "unit": "states/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if mode == _lib.MODE_FAST else "f64",
            "precision": ("tensor-core leg: split-fp16 operands (22-bit), f32 accumulation, MUFU gates; "
                          "features bit-exact except f13/f15 (big-integer logarithms) to float accuracy "
                          "before the f32 rounding; V within 1e-4 of the exact fp64 leg (max rel in "
                          "exact_leg.fast_vs_exact_max_rel), which is bit-identical to the reference"
                          if mode == _lib.MODE_FAST else "exact fp64 leg, bit-identical to the reference"),
            "data": "synthetic",
            "config": {"workload": "vgg16 synthetic scoring sweep: random partial schedules "
                                   "(SearchRng walk), v0.ckpt", "pipeline": "vgg16", "T": T,
                       "states_per_gpu": M, "mean_depth": float(depths.mean()),
                       "mode": args.mode, "l2": "inputs larger than L2 (records "
                       f"{n_records * 16 / 1e6:.0f} MB/GPU)", "parallelism": f"shard{world}"},
            "e2e": {"value": e2e_value, "unit": "states/s",
                    "h2d_bytes_per_step": e2e_h2d, "wire_format": wire_name,
                    "d2h_bytes_per_step": int(8 * M)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "greedy_wall_s": greedy,
            "beam_wall_s": beam,
            "v_callable_reference_states": level1,
            "sweep_states_per_s": sweep,
            "exact_leg": exact_leg,
            "sweep_1e8_one_gpu": big,
            "v_training": train_line,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
