#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
WDD_NVCC_EXTRA="-DWDD_LEAN=1" WDD_LIB_OUT=/tmp/libwdd_lean.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || exit 1
WDD_LIB=/tmp/libwdd_lean.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
j() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"; }
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j base
for mf in 32 16 8; do WDD_PROJ_MIN_FRAMES=$mf WDD_LIB=/tmp/libwdd_lean.so python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j lean_mf$mf; done
WDD_LIB=/tmp/libwdd_lean.so python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch 16384 2>/dev/null | j lean_single
