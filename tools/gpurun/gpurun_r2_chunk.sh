# e2e host pipeline: chunk size sweep (params per chunk)
cd $GRAFT_REPO_ROOT
for c in 33554432 16777216 67108864 134217728 33554432; do
  timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 3 --e2e-steps 4 --e2e-chunk $c 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('chunk $c', round(e['ms_per_step'],1), 'ms', round(e['value']/1e9,3), 'Gparam/s')"
done
