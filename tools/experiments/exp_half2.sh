# Hermitian half-plane FFT flush: the whole GPU suite, then each workload's bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/half_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|FAILED" gpurun_out/half_pytest.log | tail -8
for c in medium large box live; do
  st=$([ $c = medium ] && echo 300 || ([ $c = box ] && echo 20 || echo 40))
  timeout 400 python bench.py --config $c --steps $st --no-cpu-baseline --e2e-steps 1 > gpurun_out/h_$c.json 2>gpurun_out/h_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/h_$c.json'))
print('$c', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'proj %.3f'%d['roofline']['frac'], 'rd', d['latency']['readout_us']['p50'])" || tail -3 gpurun_out/h_$c.err
done
