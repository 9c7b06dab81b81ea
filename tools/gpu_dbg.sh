mkdir -p gpurun_out
timeout 300 python tools/cta0_timeline.py 1600 > gpurun_out/timeline.txt 2>&1; echo tl $?
cat gpurun_out/timeline.txt
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_srv.json 2> gpurun_out/bench_srv.err; echo bench-srv $?
tail -3 gpurun_out/bench_srv.err
tail -1 gpurun_out/bench_srv.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline']['avg_launch_us'], d['prescan'], d['phases_us_per_scan_launch'])"
timeout 1700 python -m pytest tests -m gpu -x -q --timeout 900 --durations=3 > gpurun_out/gputests.log 2>&1; echo tests $?
tail -4 gpurun_out/gputests.log
