python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/t.log
KB_GRAPH=1 python tools/kbench.py --levels 2 > gpurun_out/kb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_half_sweep_cp -c 1 -o gpurun_out/prof_cp python tools/kbench.py --levels 2 > gpurun_out/ncu.log 2>&1
