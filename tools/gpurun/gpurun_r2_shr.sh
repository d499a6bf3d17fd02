# K4 fp32 epilogue staging: generic (LD/ST.E) vs explicit shared-memory accesses
cd $GRAFT_REPO_ROOT
for v in gen shr gen shr; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 600 python bench.py --workload linear --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['per_phase_ms']; print('$v', 'fwd', round(p['fwd'],4), 'dgrad', round(p['dgrad'],4), 'wgrad', round(p['wgrad'],4), 'sm', d['clocks']['sm_mhz'])"
done
COAT_LIB=build_ab/shr/libcoat.so timeout 600 python -m pytest tests/test_gpu_linear.py -q -x 2>&1 | tail -1
COAT_LIB=build_ab/shr/libcoat.so timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -c 1 -o gpurun_out/r2/gemm_shr python tools/gemm_kernels.py > /dev/null 2>&1; echo "ncu rc=$?"
