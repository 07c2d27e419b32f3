# V-training throughput per gradient mode at two per-GPU batch sizes (bench.py v_training).
for B in 4096 16384; do
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-greedy --big-states 0 --no-exact --train-batch $B > gpurun_out/bt_$B.log 2>&1
python - $B <<'PY'
import json,sys
l=json.loads(open(f"gpurun_out/bt_{sys.argv[1]}.log").read().strip().splitlines()[-1])["v_training"]
print(sys.argv[1], "tcf", round(l["value"]/1e6,2), "M/s", round(l["ms_per_step"],4), "ms", l["tensor"]["frac"], "| tc", round(l["tc_weight_grads_only"]["value"]/1e6,2), "| exact", round(l["exact"]["value"]/1e6,2), l["holdout_mse_log"], l["exact"]["holdout_mse_log"])
PY
done
