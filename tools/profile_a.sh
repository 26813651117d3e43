set -u
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?"
for k in k_half_sweep_band k_residual_restrict_red; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_$k python tools/kbench.py --levels 2 > gpurun_out/ncu_$k.log 2>&1
  echo "ncu full $k rc=$?"
done
ls -la gpurun_out
