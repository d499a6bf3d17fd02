# K4 epilogue write spreading for the fp32 outputs only (default 20 ns per k-block) vs off: bench A/B, parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for i in 1 2 3; do for P in 0 20; do
COAT_GEMM_EPI_PAUSE_PER_KB=$P timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_pause.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_pause.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('per_kb=$P', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate x%.3f' % d['mlp_upgate']['speedup'], d['clocks']['sm_mhz'])"
done; done
timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py -q -x -k "linear or cluster or single_cta" > gpurun_out/r2/t_pause.log 2>&1; echo "linear rc=$?"; tail -1 gpurun_out/r2/t_pause.log
