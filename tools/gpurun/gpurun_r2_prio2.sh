# cfg2 graph: per-tensor records on a high-priority branch, branch-count sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for i in 1 2; do
for cfg in "rr 0 3" "pt1 1 2" "pt1 1 3" "pt1 1 4"; do set -- $cfg
COAT_BENCH_MGAQ_PLAN=$1 COAT_BENCH_MGAQ_PRIO=$2 timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-branches $3 > gpurun_out/r2/bench_mgaq_prio.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_mgaq_prio.json').read().strip().splitlines()[-1]); print('plan=$1 prio=$2 nb=$3', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
# DRAM traffic of the whole graph under the candidate plan
COAT_BENCH_MGAQ_PLAN=pt1 COAT_BENCH_MGAQ_PRIO=1 timeout -s KILL 600 ncu --nvtx --nvtx-include cfg2_layer/ --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python bench.py --workload mgaq --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r2/mgaq_graph_dram_pt1prio.csv 2>/dev/null; echo ncu rc=$?
grep -E "dram__bytes|gpu__time" gpurun_out/r2/mgaq_graph_dram_pt1prio.csv | awk -F'","' '{print $(NF-2), $NF}'
