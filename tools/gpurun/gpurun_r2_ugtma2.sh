# K4 staged gate/up epilogue: full parity (pair, 1-CTA, cluster modes), producers, sanitizer epi cases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_producers.py tests/test_gpu_k1_layouts.py tests/test_gpu_sanitizer.py -q -k "linear or upgate or producer or rms or silu or cluster or single_cta or epi or gemm" > gpurun_out/r2/t_ugtma2.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/r2/t_ugtma2.log
