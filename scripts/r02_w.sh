#!/bin/bash
# planner regret on the current build: every configuration vs the auto pick (rc paper-sweep shapes + rr list)
O=gpurun_out/r02w
mkdir -p $O
SH=$(python -c "
import json; d=json.load(open('profiles/r01_tune_rc50.json')); print(' '.join(list(d)[:30]))")
timeout 2400 python scripts/tune_sweep.py --rc $SH > $O/tune_rc.txt 2>&1
cp gpurun_out/tune_sweep.json $O/tune_rc.json
timeout 1800 python scripts/tune_sweep.py > $O/tune_rr.txt 2>&1
cp gpurun_out/tune_sweep.json $O/tune_rr.json
ls -la $O
