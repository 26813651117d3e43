# Round-2 ncu captures (run on the GPU box via gpurun; outputs in gpurun_out/):
# the fine-level kernels of the configs[3] block at 2048^2 x 128 that the
# round-1 profiles did not cover -- the red-only restriction, the black-only
# prolongation k_prolong_w<2, 2> the solve runs, and the variable-coefficient
# band sweep.  Each capture is ~20 MB (gpurun copies back <= 64 MiB).
set -u
mkdir -p gpurun_out
KB="python tools/kbench.py --nx 2048 --levels 2 --no-solve"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_prolong_w<\(int\)2, \(int\)2>' -c 1 -o gpurun_out/r02_c_prolong_w22 $KB > gpurun_out/ncu_pw.log 2>&1
echo "prolong rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_residual_restrict_red -c 1 \
    -o gpurun_out/r02_c_rr $KB > gpurun_out/ncu_rr.log 2>&1
echo "rr rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_half_sweep_bandv -c 1 \
    -o gpurun_out/r02_c_bandv python tools/kbench.py --nx 2048 --levels 1 --variable --no-solve \
    > gpurun_out/ncu_bandv.log 2>&1
echo "bandv rc=$?"
ls -la gpurun_out
