# K4 DRAM bytes per kernel by raster group (ncu, library kernels alongside)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for G in 0 4 8 16; do
COAT_GEMM_GROUP_M=$G timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --nvtx --nvtx-include "cmp/" --csv python tools/gemm_vs_library.py > gpurun_out/r2/raster_dram_g$G.csv 2>/dev/null
echo G=$G
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2/raster_dram_g$G.csv')) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); u=h.index('Metric Unit')
for r in rows[1:]:
    print(r[k][:40], r[m], r[v], r[u])
PY
done
