# task-queue kernel variants: task size / ring slots / tasks per claim
cd $GRAFT_REPO_ROOT
for v in q32c512 q16c512 q32c384 q32s3c2m2 q32c512 q16c512 q32c384 q32s3c2m2; do
  COAT_LIB=build_ab/$v/libcoat.so COAT_MGAQ_BATCH=queue timeout 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl batch 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
done
timeout 300 python bench.py --workload mgaq --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('graph', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
