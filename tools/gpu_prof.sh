#!/bin/bash
# Profiling call (under gpurun): the projection kernels of Live / Large, the Box bench launch list
# and one Box projection launch (traffic for bench.py's roofline).  Plain run first, then ncu.
tag=${1:-r02}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
summ() { python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.sum.txt 2>&1;
         python tools/ncu_lines.py gpurun_out/$1.ncu-rep 30 > gpurun_out/$1.lines.txt 2>&1; }
for c in "live 8 3" "large 64 1"; do
  set -- $c
  timeout 300 python tools/prof_cfg.py --config $1 --rows $2 --reps 1 > gpurun_out/${tag}_plain_$1.log 2>&1 && \
  timeout 900 $NCU -k regex:project_kernel -s $3 -c 1 -o gpurun_out/${tag}_$1_project -f \
      python tools/prof_cfg.py --config $1 --rows $2 --reps 1 > gpurun_out/${tag}_ncu_$1.log 2>&1
  summ ${tag}_$1_project
done
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $B > gpurun_out/${tag}_plain_box.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_launches_box_bench.csv $B > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 $NCU -k regex:project_kernel -s 200 -c 1 -o gpurun_out/${tag}_box_project -f $B > /dev/null 2>&1
summ ${tag}_box_project
timeout 900 $NCU -k regex:"rowfft|colfft|img_|scatter" -s 4 -c 4 -o gpurun_out/${tag}_box_flush -f $B > /dev/null 2>&1
summ ${tag}_box_flush
rm -f gpurun_out/${tag}_box_*.ncu-rep gpurun_out/${tag}_large_project.ncu-rep
ls -la gpurun_out | tail -20
