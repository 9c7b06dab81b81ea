# Round-2 re-validation of the tree: GPU suite, smoke, bench, ncu evidence of the dominant kernel,
# and a launch list of the sharded admission at N=1 (where its time goes).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -1 gpurun_out/bench.json
timeout 600 python bench.py --parallel sharded --no-cpu-baseline --steps 20 > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo bench_sharded $?
tail -1 gpurun_out/bench_sharded.json | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/sharded_launches.csv python bench.py --parallel sharded --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_sharded.log 2>&1; echo ncu_sharded $?
CS_SERVER=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 1600 -c 1 -o gpurun_out/r02_admit_full python tools/ncu_admit.py --skip 1600 --n 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
CS_SERVER=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:admit_kernel -c 400 --csv --log-file gpurun_out/r02_admit_launches_dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list $?
python tools/ncu_summarize.py full gpurun_out/r02_admit_full.ncu-rep gpurun_out/r02_admit_launches_dram.csv > gpurun_out/ncu_admit_summary.json; echo summ $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
tail -1 gpurun_out/smoke.log
