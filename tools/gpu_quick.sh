timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -2
timeout 600 python tools/bench_timeline.py 2>&1 | tail -8
timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 300 -c 1 -o gpurun_out/admit_full_r01b python tools/ncu_admit.py --skip 300 --n 2 > gpurun_out/ncu_full_b.log 2>&1; echo ncu $?
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1
