# K4 warp-converged MMA issuer (elect.sync) vs the single-lane issuer (base), +- TMA-store epilogue: parity, ncu, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for L in mma mmatst; do
COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_$L.log 2>&1; echo "linear $L rc=$?"; tail -1 gpurun_out/r2/t_$L.log
done
COAT_LIB=build_ab/mma/libcoat.so timeout -s KILL 900 python -m pytest tests/test_gpu_k1_layouts.py -q -x -k "cluster or single_cta" > gpurun_out/r2/t_mma_modes.log 2>&1; echo "modes rc=$?"; tail -1 gpurun_out/r2/t_mma_modes.log
for L in base mma mmatst; do
echo "lib=$L"
COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
for i in 1 2; do for L in base mma mmatst; do
COAT_LIB=build_ab/$L/libcoat.so timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_mma.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_mma.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('$L', {k: round(v,1) for k,v in d['tflops'].items()}, 'lib fwd/lt %.3f dgrad/cublas %.3f' % (l['fwd_vs_cublaslt'], l['dgrad_vs_cublas']), 'upgate %.4f x%.3f' % (d['mlp_upgate']['fused_ms'], d['mlp_upgate']['speedup']), d['clocks']['sm_mhz'])"
done; done
