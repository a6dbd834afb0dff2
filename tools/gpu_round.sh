#!/bin/bash
# One GPU round trip: parity tests, a bench line, the ncu launch list of the bench command and a
# full ncu capture of the projection kernel.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_round.sh [tag] [what...]    what in {test, bench, launches, full, smoke}
tag=${1:-r01}; shift
what=${*:-"smoke test bench launches full"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/${tag}_build.log; exit 1; }
for w in $what; do
  case $w in
    smoke) timeout 600 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${tag}_smoke.log ;;
    test) timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${tag}_pytest.log ;;
    bench) timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/${tag}_bench.json ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
        --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
        > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches rc=$?" ;;
    full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:project_kernel -s 8 -c 1 \
        -o gpurun_out/${tag}_project_full -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
        > gpurun_out/${tag}_ncu_full.log 2>&1; echo "full rc=$?"
        timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"rowdft|flush|readout" -c 3 \
        -o gpurun_out/${tag}_accum_full -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
        > gpurun_out/${tag}_ncu_full2.log 2>&1; echo "full2 rc=$?" ;;
  esac
done
