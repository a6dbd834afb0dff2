#!/bin/bash
# End-of-round evidence (under gpurun, from the repo root): tests, smoke, the default bench line and
# the other workloads, the ncu launch list of the bench command, --set full summaries of the
# dominant kernels, the overlapped-acquisition hang hunt.  Everything lands in gpurun_out/<tag>_*;
# .ncu-rep files are summarised and deleted (gpurun_out is size-limited).
tag=${1:-r02}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
for c in medium large live; do
  timeout 600 python bench.py --config $c --steps $([ $c = medium ] && echo 400 || echo 40) --no-cpu-baseline > gpurun_out/${tag}_bench_$c.json 2>/dev/null; echo "bench $c rc=$?"
done
timeout 600 python bench.py --config live --accumulator spectrum --steps 40 --no-cpu-baseline > gpurun_out/${tag}_bench_live_spectrum.json 2>/dev/null
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_launches_box_bench.csv $B > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches rc=$?"
summ() { python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.sum.txt 2>&1;
         python tools/ncu_lines.py gpurun_out/$1.ncu-rep 30 > gpurun_out/$1.lines.txt 2>&1; rm -f gpurun_out/$1.ncu-rep; }
timeout 900 $NCU -k regex:project_kernel -s 200 -c 1 -o gpurun_out/${tag}_box_project -f $B > /dev/null 2>&1; summ ${tag}_box_project
timeout 900 $NCU -k regex:"rowfft|colfft|img_|scatter" -s 4 -c 4 -o gpurun_out/${tag}_box_flush -f $B > /dev/null 2>&1; summ ${tag}_box_flush
C="python tools/prof_cfg.py --config large --rows 256 --reps 1 --batch 65536"
timeout 300 $C > /dev/null 2>&1 && timeout 900 $NCU -k regex:project_kernel -c 1 -o gpurun_out/${tag}_large_project -f $C > /dev/null 2>&1; summ ${tag}_large_project
C="python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1"
timeout 300 $C > /dev/null 2>&1 && timeout 900 $NCU -k regex:"rgemm|project_kernel" -s 8 -c 2 -o gpurun_out/${tag}_live_kernels -f $C > /dev/null 2>&1; summ ${tag}_live_kernels
for a in "live 160 G" "large 100 G" "medium 400 G" "box 16 G"; do set -- $a
  timeout 600 python tools/hang_hunt.py $1 $2 $3 > gpurun_out/${tag}_hh_$1.txt 2>&1; echo "hang hunt $1: rc=$? $(tail -1 gpurun_out/${tag}_hh_$1.txt)"; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
echo done
