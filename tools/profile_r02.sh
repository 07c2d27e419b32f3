# Round-2 evidence: full bench line, launch list, ncu full captures of the
# dominant kernels (each command has exited 0 without ncu first).
set -x
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-greedy --no-train --big-states 0 --no-exact > gpurun_out/r02_ncu_list.log 2>&1; echo list=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name regex:"k_trc|k_train" -c 40 --csv --log-file gpurun_out/r02_launches_train.csv python tools/train_tc_probe.py 16384 exact,tc,tcf > gpurun_out/r02_ncu_train.log 2>&1; echo listtrain=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:k_featurize_rows -c 1 -o gpurun_out/r02_featurize_full python bench.py --steps 1 --warmup 3 --no-cpu --no-greedy --no-train --big-states 0 --no-exact > gpurun_out/ncu_f.log 2>&1; echo feat=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_lstm_tc" -s 1 -c 1 -o gpurun_out/r02_lstm_full python bench.py --steps 1 --warmup 3 --no-cpu --no-greedy --no-train --big-states 0 --no-exact > gpurun_out/ncu_l.log 2>&1; echo lstm=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_trc_(fwd|bwd)" -c 2 -o gpurun_out/r02_trc_full python tools/train_tc_probe.py 16384 tcf > gpurun_out/ncu_t.log 2>&1; echo trc=$?
