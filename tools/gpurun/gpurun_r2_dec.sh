# vectorized bf16 decode: exactness test, linear tests, cfg4 quant phase
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_linear.py -q -x -k "decode or linear" > gpurun_out/r2/t_dec.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2/t_dec.log
for i in 1 2; do
timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_dec.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_dec.json').read().strip().splitlines()[-1]); print(round(d['value'],1), {k: round(v,4) for k,v in d['per_phase_ms'].items()}, d['clocks']['sm_mhz'])"
done
