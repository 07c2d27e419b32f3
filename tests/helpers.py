"""Shared test helpers: rebuild states from golden keys with both the
oracle (independent restatement) and the product's host mirror."""

import numpy as np

import oracle as O
from paper_2011_14486_b200 import pipeline_ir as pi
from paper_2011_14486_b200 import schedule_space as ss


def pipeline_from(entry):
    return pi.parse_pipeline(str(entry["text"]))


def oracle_params(path):
    return O.load_checkpoint(path)


def product_states(p, keys):
    return [ss.state_from_key(p, str(k)) for k in keys]


def oracle_decisions(p, key):
    body = str(key)[len(p.name) + 1:]
    return [O.as_act(ss.parse_layer_schedule(t)) for t in body.split(";") if t]


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
