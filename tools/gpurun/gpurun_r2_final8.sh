# last full validation of the round
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/t_gpu_final8.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r2/t_gpu_final8.log
timeout 600 python bench.py > gpurun_out/r2/bench_default8.json 2>gpurun_out/r2/bench_default8.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2/bench_default8.json
timeout 600 python bench.py --impl reference > gpurun_out/r2/bench_reference8.json 2>/dev/null; echo "ref rc=$?"; tail -c 400 gpurun_out/r2/bench_reference8.json
