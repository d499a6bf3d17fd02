# tools/ab_run.sh V1 V2 ... -- run bench.py once per build_ab/V/libcoat.so (A/B of kernel variants on the GPU box)
for v in "$@"; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(f"{v:10s} {d['ms_per_step']:.3f} ms  {d['roofline']['achieved']:.0f} GB/s  frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(v, "FAILED", e, open(f"gpurun_out/ab_{v}.err").read()[-500:])
PY
done
