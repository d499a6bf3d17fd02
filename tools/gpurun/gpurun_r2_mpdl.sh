cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in mbase mpdl mbase mpdl; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload mgaq --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg2', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload mgaq-fused --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v fused', round(d['ms_per_step'],4))"
done
COAT_LIB=build_ab/mpdl/libcoat.so timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_producers.py tests/test_gpu_fuzz.py -q -x > gpurun_out/r2/t_mpdl.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2/t_mpdl.log
