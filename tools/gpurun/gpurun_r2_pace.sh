# K4 TMA-store epilogue with paced stores: sweep COAT_GEMM_EPI_PACE_NS
cd $GRAFT_REPO_ROOT
for P in 0 200 500 1000 2000; do
echo "pace=$P"
COAT_GEMM_EPI_PACE_NS=$P COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel -c 1 --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-160
done
for P in 0 500 1000 0 500 1000; do
COAT_GEMM_EPI_PACE_NS=$P COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_linear_pace.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_linear_pace.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('pace $P', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f' % l['fwd_vs_cublaslt'], d['clocks']['sm_mhz'])"
done
