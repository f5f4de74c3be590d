#!/bin/bash
# GPU box: one --set full capture of the ENUF (Eq. 12) step's hot kernels at 45^3 cells (N = 512^3)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-enuf}
NCU=/usr/local/cuda/bin/ncu
CMD="python tools/enuf_bench.py"
ENUF_CELLS=45 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ENUF_CELLS=45 $NCU --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_spread_sweep|k_fft_r2c|k_fft1024_strided|k_point_records}" -c ${COUNT:-4} -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full capture rc=$?"
tail -3 gpurun_out/${TAG}_ncu_full.log
