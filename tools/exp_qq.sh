#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"rgemm" -s 1 -c 1 -f -o gpurun_out/live_rgemm2 python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1 > gpurun_out/ncu_rg2.log 2>&1
ls -la gpurun_out/live_rgemm2.ncu-rep
