# gate/up GEMM: 8 vs 16 epilogue warps (x16 TMEM loads); parity of the 16-warp default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in u8 u16 u8 u16; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 600 python bench.py --workload linear --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); u=d['mlp_upgate']; print('$v upgate fused', round(u['fused_ms'],4), 'unfused', round(u['unfused_ms'],4), 'x', round(u['speedup'],3))"
done
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py -q -x -k "linear or single_cta" > gpurun_out/r2/t_u16.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2/t_u16.log
timeout 600 ncu --set full --clock-control none -k regex:"gemm_kernel" -c 3 -o gpurun_out/r2/gemm_u16 python tools/gemm_kernels.py > /dev/null 2>&1; echo "ncu rc=$?"
