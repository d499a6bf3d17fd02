# K4 fp32 epilogue pause: 20 vs 30 vs 40 ns per k-block (ncu + bench)
cd $GRAFT_REPO_ROOT
for P in 20 30 40; do
echo "per_kb=$P"
COAT_GEMM_EPI_PAUSE_PER_KB=$P timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep -E "1, 0, 1, 0, 2|0, 1, 1, 0, 2" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
for i in 1 2; do for P in 20 30 40; do
COAT_GEMM_EPI_PAUSE_PER_KB=$P timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/bench_p3.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_p3.json').read().strip().splitlines()[-1]); l=d['library_same_shape']; print('per_kb=$P', {k: round(v,1) for k,v in d['tflops'].items()}, 'fwd/lt %.3f' % l['fwd_vs_cublaslt'], d['clocks']['sm_mhz'])"
done; done
