for cfg in "" "PMG_NO_WRAP=1" "PMG_PROLONG_JB=1" "PMG_NO_WRAP=1 PMG_PROLONG_JB=1"; do
  env $cfg python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$cfg', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
done
python tools/pcie.py 2>&1 | tail -3
