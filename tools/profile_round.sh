set -x
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-cpu --no-greedy --no-train > gpurun_out/bench_small.log 2>&1; echo small=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-greedy --no-train > gpurun_out/ncu_list.log 2>&1; echo list=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name regex:k_train -c 60 --csv --log-file gpurun_out/launches_train.csv python bench.py --states 65536 --steps 3 --warmup 3 --no-cpu --no-greedy > gpurun_out/ncu_list_train.log 2>&1; echo listtrain=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:k_featurize_rows -c 1 -o gpurun_out/r01_featurize_full python bench.py --steps 1 --warmup 3 --no-cpu --no-greedy --no-train > gpurun_out/ncu_f.log 2>&1; echo feat=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:k_lstm_tc -s 1 -c 1 -o gpurun_out/r01_lstm_full python bench.py --steps 1 --warmup 3 --no-cpu --no-greedy --no-train > gpurun_out/ncu_l.log 2>&1; echo lstm=$?
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_train_fb_group<1>" -c 1 -o gpurun_out/r01_train_tc_full python bench.py --states 65536 --steps 3 --warmup 3 --no-cpu --no-greedy > gpurun_out/ncu_t.log 2>&1; echo train=$?
