cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in base pdl base pdl; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload cfg1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg1 us', round(d['us_per_step'],2), 'frac', round(d['roofline']['frac'],4))"
done
for v in base pdl; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-extra --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v 7b', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
COAT_LIB=build_ab/pdl/libcoat.so timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fuzz.py tests/test_gpu_step_host.py tests/test_gpu_zero_p2p.py -q -x -k "not ipc and not peer" > gpurun_out/r2/t_pdl.log 2>&1; echo "pdl tests rc=$?"; tail -2 gpurun_out/r2/t_pdl.log
