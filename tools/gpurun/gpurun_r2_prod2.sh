cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"rms|silu|quant|amax" -c 14 --csv python bench.py --workload mgaq-fused --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep -E "gpu__time|inst_executed" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    print(r[0], r[4].split('(')[0][-40:], r[-3], r[-1])"
