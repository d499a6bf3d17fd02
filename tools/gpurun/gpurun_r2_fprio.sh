# fused-producer layer graph: which branch (if any) at high priority
cd $GRAFT_REPO_ROOT
for i in 1 2; do for B in "" 0 2 3; do
COAT_BENCH_FUSED_PRIO=$B timeout -s KILL 300 python bench.py --workload mgaq-fused --no-cpu-baseline > gpurun_out/bench_fp.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_fp.json').read().strip().splitlines()[-1]); print('prio=${B:-none}', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
