# quantizing GEMM epilogues: parity tests + cfg4 bench line (with the fused upgate comparison)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_linear.py -q -x > gpurun_out/r2/t_linear.log 2>&1; echo "linear tests rc=$?"
tail -30 gpurun_out/r2/t_linear.log
timeout 600 python bench.py --workload linear --no-cpu-baseline > gpurun_out/r2/bench_linear.json 2> gpurun_out/r2/bench_linear.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2/bench_linear.json; tail -5 gpurun_out/r2/bench_linear.err
