mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAIL
for c in medium live box large; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/lat_$c.json 2> gpurun_out/lat_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/lat_$c.json'));print('$c', '%.4g'%d['value'], json.dumps(d['latency']['isolated_batch_us']), 'p50', d['latency']['ingest_batch_us']['p50'])" || tail -5 gpurun_out/lat_$c.err
done
