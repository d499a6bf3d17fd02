# cfg2 (priority plan): L2 keep window sweep, time + whole-graph DRAM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for i in 1 2; do for K in 80 96 110; do
COAT_L2_KEEP_MB=$K timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline > gpurun_out/bench_keep.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_keep.json').read().strip().splitlines()[-1]); print('keep=$K', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
for K in 96 110; do
COAT_L2_KEEP_MB=$K timeout -s KILL 600 ncu --nvtx --nvtx-include cfg2_layer/ --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv python bench.py --workload mgaq --no-cpu-baseline --steps 1 --warmup 3 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print "keep='$K'", $(NF-2), $NF}'
done
