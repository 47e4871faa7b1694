#!/bin/bash
# driver-like sequence on a fresh box: build, GPU tests, smoke, default bench line, reference arm
O=gpurun_out/driver_check
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); print('build ok')" > $O/build.log 2>&1; tail -1 $O/build.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; python scripts/show_bench.py $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err; cut -c1-200 $O/ref.json
