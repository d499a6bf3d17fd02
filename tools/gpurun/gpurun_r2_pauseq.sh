# K4 quantizing epilogues (1x16 forward, gate/up): pause sweep under ncu
cd $GRAFT_REPO_ROOT
for P in 0 10 20 40 80; do
echo "q_per_kb=$P"
COAT_GEMM_EPI_PAUSE_Q_PER_KB=$P timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel --csv python tools/gemm_kernels.py 2>/dev/null | grep gemm_kernel | grep "1, 0, 1, [23], 2" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(CUtensorMap_st, CUtensorMap_st, CUtensorMap_st, Params)//' | cut -c1-120
done
