# Round-2 evidence after the FAST-leg log features (f13/f15 to float accuracy):
# GPU suite, bench line, launch list and full captures of the sweep kernels
# (each ncu command only after the same command exited 0 without ncu).
set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02b_tests.log 2>&1; echo tests=$?
timeout 900 python bench.py --no-train --no-greedy --no-cpu --big-states 0 > gpurun_out/r02b_bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-greedy --no-train --big-states 0 --no-exact > gpurun_out/r02b_ncu_list.log 2>&1; echo list=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:k_featurize_rows -c 1 -o gpurun_out/r02b_featurize_full python bench.py --steps 1 --warmup 3 --no-cpu --no-greedy --no-train --big-states 0 --no-exact > gpurun_out/ncu_fb.log 2>&1; echo feat=$?
