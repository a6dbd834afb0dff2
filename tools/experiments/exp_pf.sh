# y-FFT L2 prefetch of the output-stage rows with the half plane: Box / Large bench and ncu DRAM bytes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for c in box large; do for v in 1 0; do
  st=$([ $c = box ] && echo 20 || echo 40)
  WDD_COLFFT_PF=$v timeout 400 python bench.py --config $c --steps $st --no-cpu-baseline --e2e-steps 1 > gpurun_out/pf.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/pf.json'))
print('$c pf=$v', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'rd', d['latency']['readout_us']['p50'])"
done; done
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
for v in 1 0; do
WDD_COLFFT_PF=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rowfft|colfft" -s 2 -c 2 --csv $B 2>/dev/null | grep -E "rowfft|colfft" | awk -F'","' '{print "pf='$v'", substr($5,1,20), $(NF-2), $NF}'
done
