# K4 epilogue pacing by main-loop progress (COAT_GEMM_EPI_PACE) x store kind (STG build "stg", TMA-store build "tst")
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for L in stg tst; do
COAT_GEMM_EPI_PACE=1 COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_pace_$L.log 2>&1; echo "linear tests $L paced rc=$?"; tail -1 gpurun_out/r2/t_pace_$L.log
done
COAT_GEMM_EPI_PACE=1 COAT_GEMM_CTA=4 COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_pace_c4.log 2>&1; echo "linear tests tst paced cta4 rc=$?"; tail -1 gpurun_out/r2/t_pace_c4.log
COAT_GEMM_EPI_PACE=1 COAT_GEMM_CTA=1 COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x -k "not 8192" > gpurun_out/r2/t_pace_c1.log 2>&1; echo "linear tests tst paced cta1 rc=$?"; tail -1 gpurun_out/r2/t_pace_c1.log
for L in stg tst; do for P in 0 1; do
echo "lib=$L pace=$P"
COAT_GEMM_EPI_PACE=$P COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done; done
for i in 1 2; do for L in stg tst; do for P in 0 1; do
COAT_GEMM_EPI_PACE=$P COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_pace.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_pace.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('$L pace=$P', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate %.4f' % d['mlp_upgate']['fused_ms'], d['clocks']['sm_mhz'])"
done; done; done
