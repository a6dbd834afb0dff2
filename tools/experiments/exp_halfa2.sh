python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "projection or large or knobs or overlap" > gpurun_out/ha_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ha_pytest.log; grep -E "^FAILED|^E " gpurun_out/ha_pytest.log | head -5
for c in large; do
  timeout 300 python bench.py --config $c --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ha.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ha.json'))
print('$c', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'proj %.3f'%d['roofline']['frac'])"
done
