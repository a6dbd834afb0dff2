python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity or knobs or fullsize or spectrum or combine or shards or overlap or edge" > gpurun_out/fu_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fu_pytest.log; grep -E "^FAILED|^E  " gpurun_out/fu_pytest.log | head -10
for c in medium large; do for f in 1 0; do
  WDD_FUSED=$f timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fu.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/fu.json'));k=d['kernels_isolated']
print('$c fused=$f', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'flush', k['flush']['ms_per_launch'], 'rowdft', k['rowdft']['ms_per_launch'], 'readout', d['latency']['readout_us']['p50'])"
done; done
