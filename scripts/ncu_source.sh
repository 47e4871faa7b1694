# Dev: per-SASS-line instruction counts / stall samples of one of our kernels (source page CSV).
# usage: ncu_source.sh M N K lay tile_n cg tag
mkdir -p gpurun_out/ncu
ncu --set full --import-source on --clock-control none -c 1 -k regex:ge_fused -o /tmp/src_$7 \
    python scripts/one_call.py $1 $2 $3 $4 $5 $6 1 > /dev/null 2>&1
ncu -i /tmp/src_$7.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/src_$7.csv
ncu -i /tmp/src_$7.ncu-rep --page raw --csv > gpurun_out/ncu/raw_$7.csv
