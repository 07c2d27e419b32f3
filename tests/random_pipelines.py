"""Seeded random pipelines in the reference's text format (pipeline_ir.py
grammar): a DAG of 2-6 stages, 1-3 pure and 0-2 reduction dims each, access
maps with strides 1-2, windows 1-3 and constant entries, producer extents
set to the hull of their consumers' footprints (computed from the output
backwards).  Used by the parity tests to go beyond the checked-in
networks."""

import random

_DIMS = "xyzw"


def random_pipeline_text(seed: int, big: bool = False) -> str:
    """big: 6-12 stages, output extents up to 4096 and longer reductions, so
    anchor chains reach invocation counts past 2^64."""
    rng = random.Random(seed)
    n = rng.randint(6, 12) if big else rng.randint(2, 6)
    names = [f"s{i}" for i in range(n)]
    # stage shapes (extents of non-output stages are filled in later)
    pure = {nm: [(d, None) for d in _DIMS[: rng.randint(1, 3)]] for nm in names}
    rexts = [3, 5, 7, 16] if big else [2, 3, 4]
    red = {nm: [(f"r{k}", rng.choice(rexts)) for k in range(rng.choice([0, 0, 1, 2]))] for nm in names}
    out = names[-1]
    oexts = [64, 256, 1024, 4096] if big else [8, 16, 32, 64]
    pure[out] = [(d, rng.choice(oexts)) for d, _ in pure[out]]
    # inputs: every stage reads one or two earlier stages and maybe a buffer;
    # every stage but the output is read by some later stage
    inputs = {nm: [] for nm in names}
    for i in range(1, n):
        if big:  # a chain (plus a skip edge now and then): long anchor chains
            inputs[names[i]] = [names[i - 1]] + ([names[i - 2]] if i >= 2 and rng.random() < 0.2 else [])
        else:
            k = rng.randint(1, min(2, i))
            inputs[names[i]] = rng.sample(names[:i], k)
    for j in range(n - 1):
        if not any(names[j] in inputs[names[i]] for i in range(j + 1, n)):
            inputs[names[rng.randint(j + 1, n - 1)]].append(names[j])
    buffers = []
    for i, nm in enumerate(names):
        if i == 0 or rng.random() < 0.3:
            b = f"b{i}"
            buffers.append((b, rng.randint(1, 3)))
            inputs[nm].append(b)
    bdims = dict(buffers)
    # maps, consumers before producers so producer extents can be hulled
    maps = {}
    need = {}  # producer -> per-dim max footprint
    for nm in reversed(names):
        if nm != out:
            ext = need.get(nm, [])
            pure[nm] = [(d, max(ext[k] if k < len(ext) else 1, 1)) for k, (d, _) in enumerate(pure[nm])]
        cvars = pure[nm] + red[nm]
        for src in inputs[nm]:
            arity = bdims[src] if src in bdims else len(pure[src])
            clauses, foot = [], []
            for _ in range(arity):
                if rng.random() < 0.15:
                    w = rng.randint(1, 3)
                    clauses.append(f"_*0+{w}")
                    foot.append(w)
                else:
                    v, e = rng.choice(cvars)
                    st, w = rng.choice([1, 1, 1, 2]), rng.choice([1, 1, 2, 3])
                    clauses.append(f"{v}*{st}+{w}")
                    foot.append(st * (e - 1) + w)
            maps.setdefault(nm, []).append((src, clauses))
            prev = need.get(src, [0] * arity)
            need[src] = [max(a, b) for a, b in zip(prev, foot)]
    lines = [f"pipeline rp{'big' if big else ''}{seed}"]
    for b, ar in buffers:
        ext = need.get(b, [1] * ar)
        lines.append(f"buffer {b} dims {'x'.join(str(max(e, 1)) for e in ext)} elem {rng.choice([1, 2, 4])}")
    for nm in names:
        dims = ",".join(f"{d}:{e}" for d, e in pure[nm])
        rd = (" reduce " + ",".join(f"{d}:{e}" for d, e in red[nm])) if red[nm] else ""
        tail = " output" if nm == out else ""
        lines.append(f"stage {nm} dims {dims}{rd} flops {rng.randint(1, 20)}{tail}")
        for src, clauses in maps.get(nm, []):
            lines.append(f"  in {src} map {', '.join(clauses)}")
    return "\n".join(lines) + "\n"
