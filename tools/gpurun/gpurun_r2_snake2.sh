# snake raster default: GEMM parity in all modes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py -q -k "linear or cluster or single_cta" > gpurun_out/r2/t_snake.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/r2/t_snake.log
