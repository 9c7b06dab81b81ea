# Re-capture the dominant kernel's ncu evidence for the current sources (src_sha16) and the bench
# line that cites it; smoke.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
CS_SERVER=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 1600 -c 1 -o gpurun_out/r02_admit_full -f python tools/ncu_admit.py --skip 1600 --n 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
CS_SERVER=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:admit_kernel -c 400 --csv --log-file gpurun_out/r02_admit_launches_dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list $?
python tools/ncu_summarize.py full gpurun_out/r02_admit_full.ncu-rep gpurun_out/r02_admit_launches_dram.csv > gpurun_out/ncu_admit_summary.json; echo summ $?
cp gpurun_out/ncu_admit_summary.json profiles/ncu_admit_summary.json
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench $?
tail -1 gpurun_out/r02_bench.json | cut -c1-200
