# K4: pipeline stages of the CTA-pair GEMM and 8 epilogue warps on the coalesced fp32 epilogue
cd $GRAFT_REPO_ROOT
for v in s6 s5 s5e8 s4 s6 s5 s5e8 s4; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 600 python bench.py --workload linear --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['per_phase_ms']; print('$v', 'fwd', round(p['fwd'],4), 'dgrad', round(p['dgrad'],4), 'wgrad', round(p['wgrad'],4), 'sm', d['clocks']['sm_mhz'])"
done
COAT_LIB=build_ab/s5e8/libcoat.so timeout 600 python -m pytest tests/test_gpu_linear.py -q -x -k "not 8192" 2>&1 | tail -1
