"""Golden beam-search fixtures from the UNMODIFIED reference (oracle/_ref).

search.beam_search(prefix, model_value(v0), width) (search.py:115-133) on
the toy/deep assets, crp2d, VGG-16 and ResNet-18: width 8 (the default, and
learner.RoundConfig.beam_width) from the initial state, widths 1/3 on the
small pipelines, and width 8 from mid-schedule prefixes (the learner's
completions, learner.py:241).  Records the final schedule, the predicted V
(hex) and the reference's wall time.  One process per case.

  python tools/make_golden_beam.py   -> tests/golden/beam.json
"""

import json
import multiprocessing as mp
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"


def case_list():
    toys = ["ref:pipelines/toys/t3_chain.pl", "ref:pipelines/toys/t5_diamond.pl",
            "ref:pipelines/deep/p12_deep.pl", "assets/pipelines/nets/crp2d.pl"]
    out = []
    for f in toys:
        for w in (1, 3, 8):
            out.append((f, w, 0))
        out.append((f, 8, 2))  # from a 2-decision prefix
    out += [("assets/pipelines/nets/vgg16.pl", 8, 0), ("assets/pipelines/nets/vgg16.pl", 8, 17),
            ("assets/pipelines/nets/resnet18.pl", 8, 0), ("assets/pipelines/nets/resnet18.pl", 4, 30),
            ("assets/pipelines/nets/mobilenet_v2.pl", 8, 0), ("assets/pipelines/nets/resnet50.pl", 8, 0)]
    return out


def key_of(f, width, plen):
    return f"{f}|w{width}|p{plen}"


def path_of(f):
    return REF / "assets" / f[4:] if f.startswith("ref:") else ROOT / f


def run(case):
    f, width, plen = case
    sys.path.insert(0, str(REF))
    from tensched.pipeline_ir import parse_pipeline
    from tensched.schedule_space import apply, candidate_actions, initial_state
    from tensched.search import SearchRng, beam_search, model_value
    from tensched.value_model import load, predict
    params = load(str(ROOT / "tests" / "golden" / "v0.ckpt"))
    text = path_of(f).read_text()
    p = parse_pipeline(text)
    s = initial_state(p)
    rng = SearchRng(1000 + plen)
    for _ in range(plen):  # prefix: a seeded walk (the learner's rollouts are prefixes too)
        c = candidate_actions(s)
        s = apply(s, c[rng.randrange(len(c))])
    prefix = [d.render() for d in s.decisions]
    t0 = time.perf_counter()
    best = beam_search(s, model_value(params), width)
    wall = time.perf_counter() - t0
    return {"file": f, "text": text, "width": width, "prefix": prefix,
            "schedule": [d.render() for d in best.decisions],
            "predicted": predict(params, best).hex(), "reference_wall_s": wall}


def main():
    """--missing: only the cases not yet in beam.json (the slow ones can be
    added without recomputing the rest)."""
    path = ROOT / "tests" / "golden" / "beam.json"
    cases = case_list()
    old = {}
    if "--missing" in sys.argv and path.exists():
        old = json.loads(path.read_text())
        cases = [c for c in cases if key_of(*c) not in old]
    with mp.get_context("spawn").Pool(max(1, min(8, len(cases)))) as pool:
        res = pool.map(run, cases)
    out = dict(old)
    out.update({key_of(r["file"], r["width"], len(r["prefix"])): r for r in res})
    path.write_text(json.dumps(out, indent=0) + "\n")
    for k, r in out.items():
        print(k, round(r["reference_wall_s"], 2), "s")


if __name__ == "__main__":
    main()
