python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "projection or large or overlap or fullsize" 2>&1 | tail -2
for c in large medium box; do
  timeout 300 python bench.py --config $c --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/l5_$c.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/l5_$c.json'))
print('$c', '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'step frac %.3f'%d['step_roofline']['frac'], 'proj frac %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['share_of_step'], d['latency']['ingest_batch_us'])"
done
