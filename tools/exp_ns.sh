#!/bin/bash
# ring-depth experiment for the projection kernel + per-kernel times of the default build
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/profile_ingest.py --config medium --batches 32 --batch 512 --reps 3 --synthetic-counts 2>&1 | tail -2
for ns in 4 6; do
  WDD_NVCC_EXTRA="-DWDD_NS=$ns" WDD_LIB_OUT=/tmp/libwdd_ns$ns.so python -m paper_2212_01309_b200.build > /dev/null 2>&1
  for b in 512 8192; do echo "NS=$ns batch=$b"; WDD_LIB=/tmp/libwdd_ns$ns.so python tools/profile_ingest.py --config medium --batches $((16384/b)) --batch $b --reps 2 --synthetic-counts 2>&1 | tail -2 | head -1; done
done
python bench.py --steps 100 --no-cpu-baseline > gpurun_out/r01c_bench.json 2>&1; tail -c 1500 gpurun_out/r01c_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fft|readout|conj|flush|rowdft" -c 12 python tools/profile_ingest.py --config medium --batches 32 --batch 512 --reps 2 --synthetic-counts > gpurun_out/r01c_ncu_fft.txt 2>&1
grep -E "fft|readout|conj|duration|bytes" gpurun_out/r01c_ncu_fft.txt | head -60
