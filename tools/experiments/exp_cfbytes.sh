# y-FFT DRAM bytes: half plane on / off, prefetch on / off (Box bench flush)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read_lookup_miss.sum
for e in "WDD_HALF=1 WDD_COLFFT_PF=1" "WDD_HALF=0 WDD_COLFFT_PF=1" "WDD_HALF=0 WDD_COLFFT_PF=0" "WDD_HALF=1 WDD_COLFFT_PF=0" "WDD_HALF=1 WDD_COLFFT_TPC=1"; do
env $e timeout 900 ncu --metrics $M --clock-control none -k regex:"colfft" -s 1 -c 1 --csv $B 2>/dev/null | grep -E "colfft" | awk -F'","' '{print "'"$e"'", $(NF-2), $NF}'
done
