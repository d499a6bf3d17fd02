# cfg2 graph plans: round robin vs per-tensor records on one branch, with / without high priority
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for i in 1 2; do
for cfg in "rr 0" "pt1 0" "pt1 1" "pt2 1"; do set -- $cfg
COAT_BENCH_MGAQ_PLAN=$1 COAT_BENCH_MGAQ_PRIO=$2 timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline > gpurun_out/r2/bench_mgaq_prio.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_mgaq_prio.json').read().strip().splitlines()[-1]); print('plan=$1 prio=$2', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
