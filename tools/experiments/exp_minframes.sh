python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mf in default 8 24 32 48 64; do
  if [ $mf = default ]; then unset WDD_PROJ_MIN_FRAMES; else export WDD_PROJ_MIN_FRAMES=$mf; fi
  timeout 300 python bench.py --config medium --steps 300 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mf.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/mf.json'))
print('$mf', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'proj %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['share_of_step'])"
done
