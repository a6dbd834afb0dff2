#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01v_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_kernel -s 40 -c 1 -o gpurun_out/r01v_project_full -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowfft|colfft|img_" -c 4 -o gpurun_out/r01v_accum_full -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "full2 rc=$?"
