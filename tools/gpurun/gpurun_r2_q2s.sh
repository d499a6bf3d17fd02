# cfg4 step with the x / W quantization chains on two streams
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for i in 1 2; do
timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_q2s.json 2>gpurun_out/r2/bench_linear_q2s.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_q2s.json').read().strip().splitlines()[-1]); print(d['value'], d['per_phase_ms'], d['clocks']['sm_mhz'])"
done
tail -3 gpurun_out/r2/bench_linear_q2s.err
