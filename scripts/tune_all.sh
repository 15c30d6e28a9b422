#!/bin/bash
OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
for mode in int f32; do
  SPDP_SWEEP=$mode timeout 300 python scripts/tune_sweep.py C2,C3 16,20,24,32 2>&1 | sed "s/^/$mode /" >> $OUT/tune.txt
done
SPDP_SWEEP=int timeout 300 python scripts/tune_sweep.py C4 32,64 2>&1 | sed "s/^/int /" >> $OUT/tune.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -n 2 $OUT/pytest.txt
