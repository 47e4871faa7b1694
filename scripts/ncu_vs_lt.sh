# Dev: ncu --set full of our 512x2 / 256x2 kernels and cuBLASLt's fused bias+ReLU kernel at square
# shapes; keeps only the raw-metric CSVs (the .ncu-rep files exceed what gpurun copies back).
N="ncu --set full --clock-control none -c 1"
mkdir -p gpurun_out/ncu
for s in ${SHAPES:-8192 4096 2048}; do
$N -k regex:ge_fused -o /tmp/ours512_$s python scripts/one_call.py $s $s $s rr 512 2 1 > /dev/null 2>&1
$N -k regex:ge_fused -o /tmp/ours256_$s python scripts/one_call.py $s $s $s rr 256 2 1 > /dev/null 2>&1
$N -k regex:nvjet -o /tmp/lt_$s python scripts/lt_call.py $s $s $s 1 > /dev/null 2>&1
for r in ours512_$s ours256_$s lt_$s; do ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/ncu/$r.csv; done
done
ls -la gpurun_out/ncu
