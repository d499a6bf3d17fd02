cd $GRAFT_REPO_ROOT
for v in pf0 pf1 pf1m2 pf0 pf1 pf1m2; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload mgaq-fused --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4))"
done
for v in pf0 pf1 pf1m2; do
COAT_LIB=build_ab/$v/libcoat.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"silu_mul_pass1" -c 1 --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep -E "gpu__time|inst_executed" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print('$v', r[-3], r[-1])"
done
