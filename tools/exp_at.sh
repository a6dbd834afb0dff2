#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
b() { python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"; }
b base; WDD_ROWFFT_PDL=1 b rowfft_pdl; b base2; WDD_ROWFFT_PDL=1 b rowfft_pdl2
WDD_PROJ_MIN_FRAMES=8 b mf8; WDD_PROJ_MIN_FRAMES=32 b mf32; WDD_PROJ_WIDE_FIRST=0 b nowide
