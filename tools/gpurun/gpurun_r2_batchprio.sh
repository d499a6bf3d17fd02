# coat_quantize_batch with the per-tensor items on a high-priority stream: parity + batch-mode timing vs graph
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_quant.py -q -x -k batch > gpurun_out/r2/t_batchprio.log 2>&1; echo "batch tests rc=$?"; tail -1 gpurun_out/r2/t_batchprio.log
for i in 1 2; do for impl in batch graph; do
timeout -s KILL 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl $impl > gpurun_out/r2/bench_mgaq_bp.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_mgaq_bp.json').read().strip().splitlines()[-1]); print('$impl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
