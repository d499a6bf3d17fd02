# cfg4 step: decodes overlapped with the forward GEMM vs inside the quant phase
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for O in 0 1; do
COAT_BENCH_CFG4_OVERLAP=$O timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_ovl.json 2>gpurun_out/bench_ovl.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_ovl.json').read().strip().splitlines()[-1]); print('overlap=$O', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['per_phase_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
tail -2 gpurun_out/bench_ovl.err
