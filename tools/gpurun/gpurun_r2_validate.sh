cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 900 python -m pytest tests/test_gpu_zero_multirank.py tests/test_gpu_cpp_compat.py tests/test_gpu_zero_step.py tests/test_zero.py -x -q > gpurun_out/r2/t_zero.log 2>&1; echo "zero rc=$?"
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q --timeout 600 > gpurun_out/r2/t_san.log 2>&1; echo "san rc=$?"
timeout 900 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"
COAT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --params 268435456 --steps 3 --warmup 3 --no-e2e > gpurun_out/r2/bench_gloo2.json 2> gpurun_out/r2/bench_gloo2.err; echo "gloo2 rc=$?"
tail -3 gpurun_out/r2/t_zero.log gpurun_out/r2/t_san.log
tail -c 600 gpurun_out/r2/bench.err
