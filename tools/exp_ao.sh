#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
b() { python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"; }
b base
for rf in 2,256 3,256 3,128 4,128 4,512; do WDD_ROWFFT=$rf b rowfft=$rf; done
for cf in 3,256 4,128 4,256 5,128 5,512; do WDD_COLFFT=$cf b colfft=$cf; done
for t in 1 2 4 8; do WDD_COLFFT_TPC=$t b tpc=$t; done
WDD_FLUSH=gemm b gemm
WDD_IMG=unfused b img_unfused
