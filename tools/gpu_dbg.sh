mkdir -p gpurun_out
for i in 1 2 3; do CS_DEBUG_PROGRESS=1 timeout 600 python -m pytest -x -q tests/test_gpu_invariants.py tests/test_gpu_scale_parity.py 2>&1 | grep -E "^E .*Error|passed|failed" | cut -c1-400 | head -3; done
timeout 1700 python -m pytest tests -m gpu -x -q --timeout 900 --durations=3 > gpurun_out/gputests.log 2>&1; echo tests $?
tail -3 gpurun_out/gputests.log
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_srv.json 2> gpurun_out/bench_srv.err; echo bench-srv $?
tail -1 gpurun_out/bench_srv.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline']['avg_launch_us'], d['prescan'], d['server'])"
