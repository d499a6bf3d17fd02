# Round-2 full validation: every GPU test, the default bench line, the gloo 2-rank bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/r2/t_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 900 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"
COAT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --params 268435456 --steps 3 --warmup 3 --no-e2e > gpurun_out/r2/bench_gloo2.json 2> gpurun_out/r2/bench_gloo2.err; echo "gloo2 rc=$?"
tail -5 gpurun_out/r2/t_gpu.log
tail -c 1500 gpurun_out/r2/bench.json
tail -c 600 gpurun_out/r2/bench.err
