# sanitizer suite incl. the two-pair multicast GEMM cluster
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout -s KILL 1800 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/r2/t_san3.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/r2/t_san3.log
grep -c "Race reported\|Error" gpurun_out/sanitizer/racecheck_gemm_COAT_GEMM_CTA4.txt; head -30 gpurun_out/sanitizer/racecheck_gemm_COAT_GEMM_CTA4.txt
