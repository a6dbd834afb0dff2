python -c "import __graft_entry__ as g; g.build()" > gpurun_out/lp_build.log 2>&1
python tools/lean_probe.py
timeout 300 python bench.py --config live --steps 10 --no-cpu-baseline > gpurun_out/lp_live_default.json 2>gpurun_out/lp_err1.txt
WDD_LIB_OUT=/tmp/libwdd_lean.so WDD_NVCC_EXTRA=-DWDD_LEAN_SMEM=115712 python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > gpurun_out/lp_build2.log 2>&1; echo build2 $?
WDD_LIB=/tmp/libwdd_lean.so python tools/lean_probe.py
WDD_LIB=/tmp/libwdd_lean.so timeout 300 python bench.py --config live --steps 10 --no-cpu-baseline > gpurun_out/lp_live_lean.json 2>gpurun_out/lp_err2.txt
for f in default lean; do python -c "
import json;d=json.load(open('gpurun_out/lp_live_$f.json'))
print('$f', '%.4g'%d['value'], 'step frac %.3f'%d['step_roofline']['frac'], 'proj frac %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['share_of_step'], d['latency']['ingest_batch_us'], d['latency']['readout_us'], d['latency']['isolated_batch_us'])"; done
