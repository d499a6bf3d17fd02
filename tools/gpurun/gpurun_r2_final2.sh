# full validation after the late-round changes (queue kernel, coalesced epilogue, ...)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/t_gpu_final2.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r2/t_gpu_final2.log
