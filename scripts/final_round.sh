#!/bin/bash
# One gpurun call at the end of a work block: smoke, GPU tests, the default bench line, the ncu
# launch list of a short bench run, and one ncu --set full capture of the headline sweep.
OUT=gpurun_out/final; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" > $OUT/status.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-rows --no-cpu --no-e2e > $OUT/ncu_bench.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:irp_lazy -s 1 -c 1 -o $OUT/irp_C5 python scripts/profile_sweep.py --irp --iters 2 > $OUT/ncu_irp.log 2>&1; echo "irp rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_sweep_u16 -s 1 -c 1 \
  -o $OUT/sweep_C2 python scripts/profile_sweep.py --config C2 --ordered --iters 2 > $OUT/ncu_full.log 2>&1; echo "full rc=$?" >> $OUT/status.txt
cat $OUT/status.txt; tail -1 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log
