# after making the small-grid row FFT PDL-launched by default: Medium/Box benches + the PDL-sensitive tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py tests/test_gpu_knobs.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in medium box medium; do
  timeout 300 python bench.py --config $c --steps $([ $c = box ] && echo 20 || echo 300) --no-cpu-baseline --e2e-steps 1 > gpurun_out/rp.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rp.json'))
print('$c', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'])"
done
timeout 600 python tools/hang_hunt.py medium 400 G 2>&1 | tail -1
