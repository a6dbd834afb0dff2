# row FFT PDL-launched on lean configurations (WDD_ROWFFT_PDL=1) vs ordinary launch
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in box large medium; do for v in 0 1 0 1; do
  WDD_ROWFFT_PDL=$v timeout 300 python bench.py --config $c --steps $([ $c = box ] && echo 20 || echo 200) --no-cpu-baseline --e2e-steps 1 > gpurun_out/rp.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rp.json'))
print('$c pdl=$v', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'])"
done; done
