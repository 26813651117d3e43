set -u
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_prolong_w -c 1 \
    -o gpurun_out/prof_k_prolong_w python tools/kbench.py --levels 2 > gpurun_out/ncu_pw.log 2>&1
echo "ncu pw rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_half_sweep_seg -c 1 \
    -o gpurun_out/prof_hs_res python tools/hs_res.py > gpurun_out/ncu_hs_res.log 2>&1
echo "ncu hs_res rc=$?"
ls -la gpurun_out
