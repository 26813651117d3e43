#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list, full ncu
# capture of the fine-level kernels.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
python bench.py $ARGS > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?"
# fine-level kernels: the first launches of each in a solve are the finest level
python tools/kbench.py --levels 2 > gpurun_out/kb.log 2>&1
for k in k_half_sweep_band k_residual_restrict_red k_prolong_w; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_$k python tools/kbench.py --levels 2 > gpurun_out/ncu_$k.log 2>&1
  echo "ncu full $k rc=$?"
done
# the red half-sweep with the fused lagged convergence residual
ncu --set full --clock-control none --import-source on -k regex:k_half_sweep_seg -c 1 \
    -o gpurun_out/prof_hs_res python tools/hs_res.py > gpurun_out/ncu_hs_res.log 2>&1
echo "ncu full hs_res rc=$?"
