# K4 epilogue write spreading: COAT_GEMM_EPI_PAUSE_PER_KB sweep (ncu + bench), then parity at the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for P in 0 8 12 20; do
echo "per_kb=$P"
COAT_GEMM_EPI_PAUSE_PER_KB=$P timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
for i in 1 2; do for P in 0 8 12 20; do
COAT_GEMM_EPI_PAUSE_PER_KB=$P timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_pause.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_pause.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('per_kb=$P', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate x%.3f' % d['mlp_upgate']['speedup'], d['clocks']['sm_mhz'])"
done; done
timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_pause.log 2>&1; echo "linear rc=$?"; tail -1 gpurun_out/r2/t_pause.log
