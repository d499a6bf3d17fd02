# K4 gate/up epilogue through staging tiles + TMA stores: parity, ncu, bench A/B vs the direct-store build (base)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_producers.py -q -x > gpurun_out/r2/t_ugtma.log 2>&1; echo "linear+producers rc=$?"; tail -2 gpurun_out/r2/t_ugtma.log
COAT_GEMM_CTA=1 timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py -q -x -k "upgate and not 8192" > gpurun_out/r2/t_ugtma1.log 2>&1; echo "upgate 1-CTA rc=$?"; tail -1 gpurun_out/r2/t_ugtma1.log
for L in base ""; do
echo "lib=${L:-new}"
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "1, 0, 1, 3, 2" | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
for i in 1 2; do for L in base ""; do
COAT_LIB=${L:+build_ab/$L/libcoat.so} timeout -s KILL 300 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear_ug.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2/bench_linear_ug.json').read().strip().splitlines()[-1]); u=d['mlp_upgate']; print('${L:-new}', 'fused %.4f unfused %.4f x%.3f' % (u['fused_ms'], u['unfused_ms'], u['speedup']), {k: round(v,1) for k,v in d['tflops'].items()}, d['clocks']['sm_mhz'])"
done; done
