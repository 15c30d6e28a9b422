#!/bin/bash
# Sweep-variant timing on one GPU: int ring vs packed-fp32 ring (SPDP_F2 groupings), C2/C3/C4.
OUT=gpurun_out/${1:-tune_f2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest_parity.txt 2>&1; echo "parity rc=$?" >> $OUT/status.txt
SPDP_SWEEP=int timeout 200 python scripts/tune_sweep.py C2 20 2>&1 | sed "s/^/int /" >> $OUT/tune.txt
for cfg in 21 31 32 41 42; do
  SPDP_SWEEP=f32 SPDP_F2=$cfg timeout 200 python scripts/tune_sweep.py C2 16,20 2>&1 | sed "s/^/f2_$cfg /" >> $OUT/tune.txt
done
timeout 100 python scripts/debug_ovf.py C2 16,20 f32 >> $OUT/tune.txt 2>&1
SPDP_SWEEP=f32 timeout 300 python scripts/tune_sweep.py C3 24,32 2>&1 | sed "s/^/f2 /" >> $OUT/tune.txt
cat $OUT/status.txt $OUT/tune.txt
