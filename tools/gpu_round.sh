set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -15
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admit_kernel -s 8 -c 1 -o gpurun_out/admit_full_r01 python tools/stress_admit.py --iters 12 > gpurun_out/ncu_full.log 2>&1; echo ncu2 $?
timeout 600 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench $?
tail -1 gpurun_out/bench_r01.json
