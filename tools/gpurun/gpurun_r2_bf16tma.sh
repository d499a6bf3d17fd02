# K4 bf16 output (dgrad) by TMA store (64B-swizzled staging): parity (all modes), sanitizer gemm, ncu + bench vs base
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py tests/test_gpu_sanitizer.py tests/test_gpu_mgaq_bwd.py -q -k "linear or dgrad or cluster or single_cta or gemm or mgaq" > gpurun_out/r2/t_bf16tma.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2/t_bf16tma.log
for L in base ""; do
echo "lib=${L:-new}"
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "0, 0, 0, 1, 2" | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
for i in 1 2; do for L in base ""; do
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_bf.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_bf.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('${L:-new}', {k: round(v,1) for k,v in d['tflops'].items()}, 'dgrad/cublas %.3f' % l['dgrad_vs_cublas'], d['clocks']['sm_mhz'])"
done; done
