"""Golden cost-oracle fixtures from the UNMODIFIED reference (oracle/_ref):
benchmark() (cost_oracle.py:313-357) of random complete schedules
(search.random_schedule with SearchRng(seed)) for every asset/net under the
default MachineModel and a non-default one.

  python tools/make_golden_cost.py  -> tests/golden/costs.json
"""

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(REF))

from tensched.cost_oracle import MachineModel, benchmark  # noqa: E402
from tensched.pipeline_ir import parse_pipeline  # noqa: E402
from tensched.schedule_space import canonical_key  # noqa: E402
from tensched.search import SearchRng, random_schedule  # noqa: E402

MACHINES = {
    "default": MachineModel(),
    "small": MachineModel(flop_cost=3, mem_byte_cost=11, cache_byte_cost=2, cache_size=4096,
                          cores=8, task_overhead=250),
}


def main():
    files = sorted((REF / "assets" / "pipelines").rglob("*.pl"))
    files += sorted((ROOT / "assets" / "pipelines" / "nets").glob("*.pl"))
    out = {"machines": {k: vars(m) if hasattr(m, "__dict__") else None for k, m in MACHINES.items()},
           "pipelines": {}}
    out["machines"] = {k: {f: getattr(m, f) for f in ("flop_cost", "mem_byte_cost", "cache_byte_cost",
                                                       "cache_size", "cores", "task_overhead")}
                       for k, m in MACHINES.items()}
    for f in files:
        p = parse_pipeline(f.read_text())
        n = 6 if len(p.stages) > 40 else 24
        rows = []
        for seed in range(1, n + 1):
            s = random_schedule(p, SearchRng(seed))
            rows.append({"key": canonical_key(s),
                         **{m: str(benchmark(s, MACHINES[m]).total_millis) for m in MACHINES}})
        out["pipelines"][p.name] = {"text": f.read_text(), "states": rows}
        print(p.name, rows[0]["default"], flush=True)
    (ROOT / "tests" / "golden" / "costs.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
