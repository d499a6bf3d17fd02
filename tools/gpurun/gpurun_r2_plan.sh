cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for cfg in "rr 3" "pt2 4" "pt2 5" "pt1 3" "rr 4" "pt2 4" "rr 3"; do
  set -- $cfg
  COAT_BENCH_MGAQ_PLAN=$1 timeout 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-branches $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
done
COAT_BENCH_MGAQ_PLAN=pt2 timeout 600 ncu --nvtx --nvtx-include "cfg2_layer/" --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv python bench.py --workload mgaq --no-cpu-baseline --steps 3 --warmup 3 --mgaq-branches 4 2>/dev/null | grep dram__ | awk -F'","' '{print $(NF-2), $NF}'
for v in sbase snew sbase snew; do
  COAT_LIB=build_ab/$v/libcoat.so timeout 300 python bench.py --workload mgaq-fused --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v fused', round(d['ms_per_step'],4))"
  COAT_LIB=build_ab/$v/libcoat.so timeout 600 python bench.py --workload linear --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); u=d['mlp_upgate']; print('$v upgate fused', round(u['fused_ms'],4), 'unfused', round(u['unfused_ms'],4))"
done
COAT_LIB=build_ab/snew/libcoat.so timeout 900 python -m pytest tests/test_gpu_producers.py tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_snew.log 2>&1; echo "snew tests rc=$?"; tail -2 gpurun_out/r2/t_snew.log
