# projection variants: default build vs WDD_LEAN=0 (full variant everywhere)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WDD_LIB_OUT=/tmp/libwdd_full.so WDD_NVCC_EXTRA=-DWDD_LEAN=0 python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > gpurun_out/l0_build.log 2>&1; echo build $?
for c in large medium box; do
  for v in default full; do
    if [ $v = full ]; then export WDD_LIB=/tmp/libwdd_full.so; else unset WDD_LIB; fi
    timeout 300 python bench.py --config $c --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/l0_${c}_$v.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/l0_${c}_$v.json'))
print('$c $v', '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'step frac %.3f'%d['step_roofline']['frac'], 'proj frac %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['share_of_step'])"
  done
done
