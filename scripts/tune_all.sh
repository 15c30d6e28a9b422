#!/bin/bash
OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
SPDP_SWEEP=deque timeout 300 python scripts/tune_sweep.py C2,C3,C4 64 2>&1 | sed "s/^/deque /" >> $OUT/tune.txt
timeout 300 python scripts/tune_irp.py >> $OUT/tune.txt 2>&1
SPDP_SWEEP=deque timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_deque.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
