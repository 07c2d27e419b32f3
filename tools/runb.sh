#!/bin/bash
# usage: runb.sh label [bench args...]; prints value/e2e/kernel_ms or the error
label=$1; shift
timeout 300 python bench.py "$@" > gpurun_out/be_$label.log 2>&1
python - "$label" <<'PY'
import json, sys
lab = sys.argv[1]
txt = open(f"gpurun_out/be_{lab}.log").read().strip().splitlines()
try:
    l = json.loads(txt[-1]); print(lab, round(l["value"]/1e6, 1), round(l["e2e"]["value"]/1e6, 1), l["roofline"]["kernel_ms"])
except Exception:
    print(lab, "FAILED:", [t for t in txt if "Error" in t or "error" in t][-2:])
PY
