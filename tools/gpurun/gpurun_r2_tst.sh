# K4 fp32 epilogue by TMA bulk-tensor stores (COAT_GEMM_TMA_STORE=1 build): parity, ncu, bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
COAT_LIB=build_ab/tst/libcoat.so timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_tst.log 2>&1; echo "linear tests (tma store) rc=$?"; tail -3 gpurun_out/r2/t_tst.log
COAT_LIB=build_ab/tst/libcoat.so COAT_GEMM_CTA=1 timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x -k "not 8192" > gpurun_out/r2/t_tst1.log 2>&1; echo "linear tests (tma store, 1 CTA) rc=$?"; tail -2 gpurun_out/r2/t_tst1.log
for L in "" build_ab/tst/libcoat.so; do
echo "lib=${L:-default}"
COAT_LIB=$L timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160
done
for L in "" build_ab/tst/libcoat.so "" build_ab/tst/libcoat.so; do
COAT_LIB=$L timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_tst.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_tst.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('${L:-default}', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f' % l['fwd_vs_cublaslt'], d['clocks']['sm_mhz'])"
done
