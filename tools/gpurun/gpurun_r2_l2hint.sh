# K4 operand-load L2 policies (COAT_GEMM_L2HINT): ncu DRAM/time per GEMM, bench A/B, parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for H in 0 1; do
echo "l2hint=$H"
COAT_GEMM_L2HINT=$H timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
for i in 1 2; do for H in 0 1; do
COAT_GEMM_L2HINT=$H timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_l2.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_l2.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('l2hint=$H', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate %.4f' % d['mlp_upgate']['fused_ms'], d['clocks']['sm_mhz'])"
done; done
COAT_GEMM_L2HINT=1 timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_l2.log 2>&1; echo "linear rc=$?"; tail -1 gpurun_out/r2/t_l2.log
