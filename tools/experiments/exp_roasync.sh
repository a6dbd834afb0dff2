# pipelined readouts (opts.readout_async): correctness tests, then bench with and without
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_overlap.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in medium box large live; do for v in 0 1; do
  st=$([ $c = medium ] && echo 300 || ([ $c = box ] && echo 20 || echo 40))
  timeout 400 python bench.py --config $c --steps $st --no-cpu-baseline --e2e-steps 1 --readout-async $v > gpurun_out/ra.json 2>gpurun_out/ra_$c$v.err
  python -c "
import json;d=json.load(open('gpurun_out/ra.json'))
print('$c async=$v', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'proj %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/ra_$c$v.err
done; done
