# ncu --set full of the Box flush kernels (half-plane row FFT + y-FFT), and the knobs test
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_knobs.py -q -p no:cacheprovider 2>&1 | tail -2
NCU="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bf_plain.json 2>&1; echo "plain rc=$?"
timeout 1200 $NCU -k regex:"rowfft|colfft" -s 2 -c 2 -o gpurun_out/bf -f $B > gpurun_out/bf_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/bf.ncu-rep > gpurun_out/bf.sum.txt 2>&1
python tools/ncu_lines.py gpurun_out/bf.ncu-rep 40 > gpurun_out/bf.lines.txt 2>&1
rm -f gpurun_out/bf.ncu-rep
