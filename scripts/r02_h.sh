#!/bin/bash
O=gpurun_out/r02h
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_pacqspin.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_configs or split_k or stream_k or batched or odd_shapes or swap or layouts_ragged or multicast or gemm2" > $O/pytest_pacqspin.log 2>&1; echo "rc=$?" >> $O/pytest_pacqspin.log
bash scripts/ab.sh $O/ab.txt spin pacq pacqspin
ls -la $O
