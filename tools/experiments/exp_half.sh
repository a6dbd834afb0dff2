# Hermitian half-plane FFT flush: the GPU suite, then benches with WDD_HALF=0 / 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/half_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/half_pytest.log
for c in medium large box live; do for v in 0 1; do
  st=$([ $c = medium ] && echo 300 || ([ $c = box ] && echo 20 || echo 40))
  WDD_HALF=$v timeout 400 python bench.py --config $c --steps $st --no-cpu-baseline --e2e-steps 1 > gpurun_out/h.json 2>gpurun_out/h_$c$v.err
  python -c "
import json;d=json.load(open('gpurun_out/h.json'))
print('$c half=$v', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'rd', d['latency']['readout_us']['p50'])" || tail -3 gpurun_out/h_$c$v.err
done; done
