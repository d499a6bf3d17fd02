# K4 tiny shapes (one partial tile everywhere) on every GEMM mode
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_linear.py -q -k "16-32" > gpurun_out/r2/t_tiny.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/r2/t_tiny.log
for C in 1 4; do COAT_GEMM_CTA=$C timeout -s KILL 600 python -m pytest tests/test_gpu_linear.py -q -k "16-32" > gpurun_out/r2/t_tiny_$C.log 2>&1; echo "cta=$C rc=$?"; tail -1 gpurun_out/r2/t_tiny_$C.log; done
