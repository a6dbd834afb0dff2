python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/hang_hunt.py live 120 G > gpurun_out/rg3_hh.txt 2>&1; echo "hang hunt rc=$? $(tail -1 gpurun_out/rg3_hh.txt)"
timeout 300 python tools/hang_hunt.py live 60 spectrum > gpurun_out/rg3_hh2.txt 2>&1; echo "hang hunt spec rc=$? $(tail -1 gpurun_out/rg3_hh2.txt)"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cadence or live or deterministic or combine or shards or tiny" > gpurun_out/rg3_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/rg3_pytest.log
for acc in G spectrum; do
timeout 300 python bench.py --config live --steps 20 --accumulator $acc --no-cpu-baseline --e2e-steps 1 > gpurun_out/rg3.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rg3.json'));k=d['kernels_isolated']
print('live $acc', '%.4g'%d['value'], 'step %.3f'%d['step_roofline']['frac'], 'flush %.3f'%k['flush']['ms_per_launch'], 'readout %.0f'%d['latency']['readout_us']['p50'])"
done
