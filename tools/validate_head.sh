nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/gputest.log 2>&1; echo pytest rc=$? >> gpurun_out/gputest.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/gputest.log; tail -1 gpurun_out/smoke.log; wc -c gpurun_out/bench.json gpurun_out/bench_ref.json gpurun_out/launches.csv
