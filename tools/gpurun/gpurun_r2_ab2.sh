# K1 A/B: wait style (K1_WAIT) x arrival style (K1_ARRIVE), ABCD twice; full GPU suite; K1 ncu capture with source
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
bash tools/abk1.sh w1a1:build_ab/w1a1/libcoat.so:8 w0a1:build_ab/w0a1/libcoat.so:8 w1a0:build_ab/w1a0/libcoat.so:8 w0a0:build_ab/w0a0/libcoat.so:8 w1a1b:build_ab/w1a1/libcoat.so:8 w0a1b:build_ab/w0a1/libcoat.so:8 w1a0b:build_ab/w1a0/libcoat.so:8 w0a0b:build_ab/w0a0/libcoat.so:8
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/t_gpu2.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r2/t_gpu2.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_ws_kernel -c 1 -o gpurun_out/r2/k1_v25 python bench.py --params 499998976 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r2/ncu_k1.log 2>&1; echo "ncu rc=$?"
