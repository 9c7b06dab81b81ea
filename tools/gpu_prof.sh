set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 300 -c 1 -o gpurun_out/r01_admit_prescan_full python tools/ncu_admit.py --skip 300 --n 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:admit_kernel -c 400 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list $?
timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; echo bench $?
tail -1 gpurun_out/r01_bench.json
