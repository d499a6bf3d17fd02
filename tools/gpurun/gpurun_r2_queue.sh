# cfg2 through coat_quantize_batch's persistent task-queue kernel vs the 3-branch graph; parity; DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_quant.py -q -x -k batch > gpurun_out/r2/t_queue.log 2>&1; echo "batch tests rc=$?"; tail -3 gpurun_out/r2/t_queue.log
for v in graph queue graph queue; do
  if [ $v = queue ]; then E="COAT_MGAQ_BATCH=queue"; I=batch; else E=""; I=graph; fi
  env $E timeout 300 python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl $I 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), d['config']['impl'])"
done
COAT_MGAQ_BATCH=queue timeout 600 ncu --cache-control none --clock-control none -k regex:mgaq_queue -c 3 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python bench.py --workload mgaq --no-cpu-baseline --mgaq-impl batch --steps 3 --warmup 3 2>/dev/null | grep -E "dram__|gpu__time" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[0], r[-3], r[-1])"
