#!/bin/bash
# End-of-round evidence (under gpurun, from the repo root): tests, the bench line, the ncu launch
# list of the bench command, --set full summaries of the dominant kernels of every workload, and
# bench_live lines.  Everything lands in gpurun_out/<tag>_*; the .ncu-rep files are summarised and
# deleted (gpurun_out is size-limited).
tag=${1:-r01}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
for c in large live box; do timeout 600 python tools/bench_live.py --config $c --reps 3 > gpurun_out/${tag}_live_$c.json 2>&1; done
timeout 600 python tools/bench_live.py --config live --reps 3 --accumulator spectrum > gpurun_out/${tag}_live_live_spectrum.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_launches_medium_bench.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches rc=$?"
summ() { python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.sum.txt 2>&1;
         python tools/ncu_hot.py gpurun_out/$1.ncu-rep 25 > gpurun_out/$1.hot.txt 2>&1; }
timeout 1200 $NCU -k regex:project_kernel -s 8 -c 1 -o gpurun_out/${tag}_medium_project -f \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
summ ${tag}_medium_project
python tools/ncu_traffic.py gpurun_out/${tag}_medium_project.ncu-rep medium > /dev/null 2>&1
cp profiles/ncu_traffic.json gpurun_out/${tag}_ncu_traffic.json
timeout 1200 $NCU -k regex:"rowfft|colfft|scatter|img_" -c 4 -o gpurun_out/${tag}_medium_flush -f \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
summ ${tag}_medium_flush
timeout 1200 $NCU -k regex:"rgemm|rowfft" -s 2 -c 2 -o gpurun_out/${tag}_live_flush -f \
    python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1 > /dev/null 2>&1
summ ${tag}_live_flush
timeout 1200 $NCU -k regex:project_kernel -s 3 -c 1 -o gpurun_out/${tag}_live_project -f \
    python tools/prof_cfg.py --config live --rows 8 --reps 1 > /dev/null 2>&1
summ ${tag}_live_project
timeout 1200 $NCU -k regex:project_kernel -s 1 -c 1 -o gpurun_out/${tag}_large_project -f \
    python tools/prof_cfg.py --config large --rows 64 --reps 1 > /dev/null 2>&1
summ ${tag}_large_project
timeout 1200 $NCU -k regex:"rowfft|colfft" -c 2 -o gpurun_out/${tag}_large_flush -f \
    python tools/prof_cfg.py --config large --rows 256 --reps 1 > /dev/null 2>&1
summ ${tag}_large_flush
rm -f gpurun_out/*.ncu-rep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
echo done
