python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
C="python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1"
timeout 300 $C > gpurun_out/rg_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgemm -s 1 -c 1 -o gpurun_out/rg_live -f $C > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/rg_live.ncu-rep > gpurun_out/rg_live.sum.txt; python tools/ncu_lines.py gpurun_out/rg_live.ncu-rep 40 > gpurun_out/rg_live.lines.txt
cat gpurun_out/rg_live.sum.txt
