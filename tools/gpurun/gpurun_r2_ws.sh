# per-call coop MGAQ workspace, per-instantiation cluster query: quant + GEMM-mode tests, MGAQ sanitizer cases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_quant.py tests/test_gpu_k1_layouts.py tests/test_gpu_sanitizer.py -q -x -k "batch or cluster or single_cta or mgaq" > gpurun_out/r2/t_ws.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/r2/t_ws.log
