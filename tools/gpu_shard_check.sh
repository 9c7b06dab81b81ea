# Sharded path: parity tests, its phase timeline, bench at N=1 (sharded) with the parity leg.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_scale_parity.py -m gpu -x -q > gpurun_out/pytest_shard.log 2>&1; echo pytest_shard $?
tail -3 gpurun_out/pytest_shard.log
timeout 600 python tools/shard_timeline.py > gpurun_out/shard_timeline.txt 2>&1; echo tl $?; tail -19 gpurun_out/shard_timeline.txt
timeout 600 python bench.py --parallel sharded --steps 20 > gpurun_out/bench_sharded_peer.json 2> gpurun_out/bench_sharded_peer.err; echo bench_sharded $?
tail -1 gpurun_out/bench_sharded_peer.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d.get('parity'))"
