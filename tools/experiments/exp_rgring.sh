# rgemm ring depths: (B ring, W/G stages per group); Live bench per variant
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { tag=$1; shift; if [ "$tag" != default ]; then WDD_LIB_OUT=/tmp/lib_$tag.so WDD_NVCC_EXTRA="$*" python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > gpurun_out/rr_$tag.log 2>&1 || { echo "$tag build failed"; tail -5 gpurun_out/rr_$tag.log; return; }; export WDD_LIB=/tmp/lib_$tag.so; else unset WDD_LIB; fi
  timeout 300 python bench.py --config live --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/rr.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rr.json'));k=d['kernels_isolated']
print('$tag', '%.4g'%d['value'], 'step frac %.3f'%d['step_roofline']['frac'], 'flush %.3f'%k['flush']['ms_per_launch'], 'readout p50 %.0f'%d['latency']['readout_us']['p50'])"; }
run default
run nb3_nwg2 -DWDD_RG_NB=3 -DWDD_RG_NWG=2
run nb4_nwg2 -DWDD_RG_NB=4 -DWDD_RG_NWG=2
run nb2_nwg2 -DWDD_RG_NB=2 -DWDD_RG_NWG=2
