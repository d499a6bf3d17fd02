# tools/abk1.sh NAME:LIB:EW ... -- K1 bench per (library, COAT_K1_EW) variant on the GPU box
for spec in "$@"; do
  IFS=: read name lib ew <<< "$spec"
  COAT_K1_EW=$ew COAT_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>gpurun_out/abk1_$name.err | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$name', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4))
except Exception as e: print('$name FAILED', e)"
done
