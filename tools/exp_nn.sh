#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/prof_cfg.py --config large --rows 64 --reps 1 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:project_kernel -s 1 -c 1 -f -o gpurun_out/large_proj python tools/prof_cfg.py --config large --rows 64 --reps 1 > gpurun_out/ncu_large.log 2>&1
$NCU -k regex:project_kernel -s 3 -c 1 -f -o gpurun_out/live_proj python tools/prof_cfg.py --config live --rows 8 --reps 1 > gpurun_out/ncu_live.log 2>&1
$NCU -k regex:"rowfft|colfft|colgemm|img_" -c 6 -f -o gpurun_out/live_flush python tools/prof_cfg.py --config live --rows 64 --reps 1 > gpurun_out/ncu_live_flush.log 2>&1
WDD_FLUSH=gemm $NCU -k regex:"colgemm" -c 1 -f -o gpurun_out/live_colgemm python tools/prof_cfg.py --config live --rows 64 --reps 1 > gpurun_out/ncu_live_cg.log 2>&1
$NCU -k regex:"rowfft|colfft|img_" -c 6 -f -o gpurun_out/large_flush python tools/prof_cfg.py --config large --rows 256 --reps 1 > gpurun_out/ncu_large_flush.log 2>&1

for r in large_proj live_proj live_flush live_colgemm large_flush; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.sum.txt 2>&1
  python tools/ncu_hot.py gpurun_out/$r.ncu-rep 25 > gpurun_out/$r.hot.txt 2>&1
  rm -f gpurun_out/$r.ncu-rep
done
