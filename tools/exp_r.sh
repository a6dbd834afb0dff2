#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
j() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"; }
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j base
python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch 16384 2>/dev/null | j single
for ns in 8; do WDD_NVCC_EXTRA="-DWDD_NS=$ns" WDD_LIB_OUT=/tmp/libwdd_ns$ns.so python -m paper_2212_01309_b200.build > /dev/null 2>&1
WDD_LIB=/tmp/libwdd_ns$ns.so python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j ns$ns
WDD_LIB=/tmp/libwdd_ns$ns.so python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch 16384 2>/dev/null | j ns${ns}single; done
