import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): print(line); continue
    d=json.loads(line)
    print("value %.4g e2e %.4g kernels %s greedy %s clocks %s" % (d["value"], d["e2e"]["value"], d["roofline"]["kernel_ms"], {k:v["wall_s"] for k,v in d.get("greedy_wall_s",{}).items()}, d["clocks"]))
