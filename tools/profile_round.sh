#!/bin/bash
# Run on the GPU box (via gpurun): smoke, bench line, then tools/profile_a.sh
# (ncu launch list + full captures of the band half-sweep and the red
# restriction).  The other two fine-level captures are tools/profile_b.sh,
# run as a separate gpurun call: gpurun copies back at most 64 MiB and each
# full capture is ~17 MB.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
bash tools/profile_a.sh
