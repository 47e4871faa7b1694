#!/bin/bash
# per-SASS-line stall samples (ncu source page) of the 2048^3 and 256^3 kernels
bash scripts/ncu_source.sh 2048 2048 2048 rr 0 0 s2048
bash scripts/ncu_source.sh 256 256 256 rr 0 0 s256
bash scripts/ncu_source.sh 35 8457 2560 rr 0 0 sskinny
ls -la gpurun_out/ncu/
head -3 gpurun_out/ncu/src_s2048.csv | cut -c1-2000
