#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3 4 5 6; do timeout 300 python tools/hang_hunt.py live 40 G > /tmp/a.txt 2>&1; echo "nwg2 rc=$? $(grep -c 'ok$' /tmp/a.txt) scans ok"; done
for acc in G spectrum; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nwg2 live $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -2 /tmp/o.txt; done
sed -i 's/^constexpr int kRgNB = 3; /constexpr int kRgNB = 2; /' paper_2212_01309_b200/csrc/kernels.cu
WDD_NVCC_EXTRA=-DWDD_RG_NWG=3 python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || echo BUILD FAIL
for i in 1 2 3; do timeout 300 python tools/hang_hunt.py live 40 G > /tmp/a.txt 2>&1; echo "nwg3 rc=$? $(grep -c 'ok$' /tmp/a.txt) scans ok"; done
for acc in G spectrum; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nwg3 live $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -2 /tmp/o.txt; done
