# cfg2 with the L2 plan (per-tensor records on one branch): bench lines for 3/4 branches and batch, whole-graph DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for B in 3 4 3 4; do
  timeout 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-branches $B 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('branches $B', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'sm', d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl batch 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('batch', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'sm', d['clocks']['sm_mhz'])"
for K in 80 1000; do
  COAT_L2_KEEP_MB=$K timeout 600 ncu --nvtx --nvtx-include "cfg2_layer/" --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python bench.py --workload mgaq --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/mgaq_graph_dram_p$K.csv 2>/dev/null; echo "ncu $K rc=$?"
  grep -E "dram__bytes|gpu__time" gpurun_out/r2/mgaq_graph_dram_p$K.csv | tail -3 | awk -F'","' '{print $(NF-2), $NF}'
done
timeout 600 python -m pytest tests/test_gpu_quant.py -q -x -k batch > gpurun_out/r2/t_quant2.log 2>&1; echo "batch tests rc=$?"; tail -2 gpurun_out/r2/t_quant2.log
