cd $GRAFT_REPO_ROOT
for v in base ctab base ctab; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload cfg1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg1 us', round(d['us_per_step'],2), 'frac', round(d['roofline']['frac'],4))"
done
bash tools/abk1.sh base7b:build_ab/base/libcoat.so:8 ctab7b:build_ab/ctab/libcoat.so:8
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_pack_prepare.py tests/test_gpu_k1_layouts.py -q -x > gpurun_out/r2/t_ctab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2/t_ctab.log
