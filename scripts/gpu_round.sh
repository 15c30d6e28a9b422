#!/bin/bash
# One gpurun call: GPU tests, bench lines, the ncu launch list and full captures.
# Usage: scripts/gpu_round.sh <tag> [phases...]
set -u
TAG=${1:-r01}; shift || true
PHASES=${@:-test bench ncu full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for p in $PHASES; do
  case $p in
    test) timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
    benchfast) timeout 600 python bench.py --no-cpu --no-rows > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/status.txt ;;
    ncu) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
           python bench.py --steps 5 --warmup 3 --no-rows --no-cpu --no-e2e > $OUT/ncu_bench.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt ;;
    full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_sweep -s 1 -c 1 \
           -o $OUT/sweep_C2 python scripts/profile_sweep.py --config C2 --iters 2 > $OUT/ncu_full.log 2>&1; echo "full rc=$?" >> $OUT/status.txt ;;
    full3) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_sweep -s 1 -c 1 \
           -o $OUT/sweep_C3 python scripts/profile_sweep.py --config C3 --iters 2 > $OUT/ncu_full3.log 2>&1; echo "full3 rc=$?" >> $OUT/status.txt ;;
    full4) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_deque -s 1 -c 1 \
           -o $OUT/sweep_C4 python scripts/profile_sweep.py --config C4 --iters 2 > $OUT/ncu_full4.log 2>&1; echo "full4 rc=$?" >> $OUT/status.txt ;;
    fullnbr) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_nbr -s 1 -c 1 \
           -o $OUT/nbr_C3 python scripts/profile_sweep.py --config C3 --nbr --iters 2 > $OUT/ncu_fullnbr.log 2>&1; echo "fullnbr rc=$?" >> $OUT/status.txt ;;
    fullgran) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_nbr -s 1 -c 1 \
           -o $OUT/nbr_gran_C3 python scripts/profile_sweep.py --config C3 --nbr --granular --iters 2 > $OUT/ncu_fullgran.log 2>&1; echo "fullgran rc=$?" >> $OUT/status.txt ;;
    fulllim) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_limits_ring -s 1 -c 1 \
           -o $OUT/limits_C2 python scripts/profile_sweep.py --config C2 --limits --iters 2 > $OUT/ncu_fulllim.log 2>&1; echo "fulllim rc=$?" >> $OUT/status.txt ;;
    fullf32) timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_f32_ring -s 1 -c 1 \
           -o $OUT/f32_C2 python scripts/profile_sweep.py --config C2 --f32 --iters 2 > $OUT/ncu_fullf32.log 2>&1; echo "fullf32 rc=$?" >> $OUT/status.txt ;;
    fullirp) timeout 900 ncu --set full --clock-control none --import-source on -k regex:irp_la -s 1 -c 1 \
           -o $OUT/irp_C5 python scripts/profile_sweep.py --irp --iters 2 > $OUT/ncu_fullirp.log 2>&1; echo "fullirp rc=$?" >> $OUT/status.txt ;;
    micro) ./scripts/micro_alu > $OUT/micro.txt 2>&1; echo "micro rc=$?" >> $OUT/status.txt ;;
  esac
done
cat $OUT/status.txt
