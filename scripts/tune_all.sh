#!/bin/bash
# sweep-kernel timing matrix over arithmetic mode x vote stride x window hint
OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
for mode in int f32; do for v in 2 4 8; do
  SPDP_SWEEP=$mode SPDP_VOTE_EVERY=$v timeout 300 python scripts/tune_sweep.py C2,C3 8,16,32 2>&1 | sed "s/^/$mode /" >> $OUT/tune.txt
done; done
SPDP_SWEEP=f32 timeout 300 python scripts/tune_sweep.py C4 32 2>&1 | sed "s/^/f32 /" >> $OUT/tune.txt
SPDP_SWEEP=int timeout 300 python scripts/tune_sweep.py C4 32,64 2>&1 | sed "s/^/int /" >> $OUT/tune.txt
for mode in int f32; do SPDP_SWEEP=$mode timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$mode.txt 2>&1; tail -1 $OUT/pytest_$mode.txt; done
