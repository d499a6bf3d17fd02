# cfg2: L2 keep budget sweep for the per-tensor re-read (bench lines) + whole-graph ncu DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for K in 1000 64 80 96 112 1000 80 96; do
  COAT_L2_KEEP_MB=$K timeout 300 python bench.py --workload mgaq --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('keep $K', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'sm', d['clocks']['sm_mhz'])"
done
for K in 1000 80 96; do
  COAT_L2_KEEP_MB=$K timeout 600 ncu --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -c 4 --csv python bench.py --workload mgaq --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/mgaq_graph_dram_$K.csv 2>gpurun_out/r2/mgaq_graph_dram_$K.err; echo "ncu $K rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_quant.py -q -x > gpurun_out/r2/t_quant.log 2>&1; echo "quant tests rc=$?"; tail -2 gpurun_out/r2/t_quant.log
