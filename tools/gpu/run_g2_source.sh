# source-level (SASS) stall sampling of the box-grid pass on config 3: 8 launches, full set
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/g2src
python tools/prof_kernels.py spmv auto > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_spmv_grid2 -s 2 -c 8 \
    -o /tmp/g2src/g2 python tools/prof_kernels.py spmv auto > gpurun_out/g2src_ncu.log 2>&1
ncu -i /tmp/g2src/g2.ncu-rep --page source --csv --print-source sass > gpurun_out/g2_source.csv 2> gpurun_out/g2_source.err
ls -la gpurun_out/g2_source.csv
head -c 1500 gpurun_out/g2_source.csv
