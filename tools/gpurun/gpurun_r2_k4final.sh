# K4 with the converged MMA issuer + TMA-store fp32 epilogue as default: GEMM tests, modes, sanitizer
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1800 python -m pytest tests/test_gpu_linear.py tests/test_gpu_k1_layouts.py tests/test_gpu_sanitizer.py -q -k "linear or cluster or single_cta or gemm or epi or upgate" > gpurun_out/r2/t_k4final.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/r2/t_k4final.log
