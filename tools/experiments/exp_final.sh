mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on"
C="python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1"
timeout 300 $C > /dev/null 2>&1 && timeout 900 $NCU -k regex:"rgemm|rowfft" -c 4 -o gpurun_out/r02f_live_flush -f $C > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02f_live_flush.ncu-rep > gpurun_out/r02f_live_flush.sum.txt 2>&1
python tools/ncu_lines.py gpurun_out/r02f_live_flush.ncu-rep 30 > gpurun_out/r02f_live_flush.lines.txt 2>&1; rm -f gpurun_out/r02f_live_flush.ncu-rep
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02f_box_rep$i.json 2>/dev/null; echo "rep $i rc=$?"; done
echo done
