cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in e4 e8 e8all e4 e8 e8all; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 600 python bench.py --workload linear --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['per_phase_ms']; u=d['mlp_upgate']; print('$v', 'fwd', round(p['fwd'],4), 'dgrad', round(p['dgrad'],4), 'wgrad', round(p['wgrad'],4), 'upgate fused', round(u['fused_ms'],4), 'unfused', round(u['unfused_ms'],4), 'sm', d['clocks']['sm_mhz'])"
done
COAT_LIB=build_ab/e8all/libcoat.so timeout 900 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_e8all.log 2>&1; echo "e8all tests rc=$?"; tail -2 gpurun_out/r2/t_e8all.log
COAT_LIB=build_ab/e8/libcoat.so COAT_GEMM_CTA=1 timeout 900 python -m pytest tests/test_gpu_linear.py -q -x -k "not 8192" > gpurun_out/r2/t_e8c1.log 2>&1; echo "e8 1cta tests rc=$?"; tail -2 gpurun_out/r2/t_e8c1.log
