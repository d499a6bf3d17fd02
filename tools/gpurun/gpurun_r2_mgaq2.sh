# cfg2 whole-layer DRAM bytes (one CUDA-graph replay, real branch concurrency) per L2 keep budget; PeerZeroAdamW test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for K in 1000 0 80; do
  COAT_L2_KEEP_MB=$K timeout 600 ncu --nvtx --nvtx-include "cfg2_layer/" --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python bench.py --workload mgaq --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2/mgaq_graph_dram_$K.csv 2>gpurun_out/r2/mgaq_graph_dram_$K.err; echo "ncu $K rc=$?"
  grep -E "dram__bytes|gpu__time" gpurun_out/r2/mgaq_graph_dram_$K.csv | tail -3
done
timeout 900 python -m pytest tests/test_gpu_zero_p2p.py -q -x -k peer > gpurun_out/r2/t_peer.log 2>&1; echo "peer tests rc=$?"; tail -30 gpurun_out/r2/t_peer.log
