python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in medium live box large; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/lat_$c.json 2>gpurun_out/lat_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/lat_$c.json'));l=d['latency']
print('$c', '%.4g'%d['value'], 'step %.3f'%d['step_roofline']['frac'], 'batch p50 %.1f'%l['ingest_batch_us']['p50'], 'iso', l['isolated_batch_us'])"
done
