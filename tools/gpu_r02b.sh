# Round-2 iteration: parity subset, the CTA-0 timeline, one bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_invariants.py -x -q --timeout 600 > gpurun_out/t_iter.log 2>&1; echo tests $?
tail -5 gpurun_out/t_iter.log
timeout 300 python tools/cta0_timeline.py 1600 > gpurun_out/timeline.txt 2>&1; echo tl $?
cat gpurun_out/timeline.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench $?
tail -1 gpurun_out/bench_iter.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step')}, d['e2e']['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['prescan'], d.get('phases_us_per_scan_launch'))"
tail -3 gpurun_out/bench_iter.err
