python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cadence or live or deterministic or combine or shards" > gpurun_out/rg2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rg2_pytest.log
timeout 300 python bench.py --config live --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/rg2.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rg2.json'));k=d['kernels_isolated']
print('live', '%.4g'%d['value'], 'step %.3f'%d['step_roofline']['frac'], 'flush %.3f'%k['flush']['ms_per_launch'], 'readout %.0f'%d['latency']['readout_us']['p50'])"
timeout 300 python tools/hang_hunt.py live 160 G > gpurun_out/rg2_hh.txt 2>&1; echo "hang hunt rc=$? $(tail -1 gpurun_out/rg2_hh.txt)"
