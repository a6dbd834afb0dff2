#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
python - <<'PY'
import paper_2212_01309_b200 as w
from synth import CONFIGS
for n in ["tiny","medium","large","live","box"]:
    c=CONFIGS[n]; p=w.Plan.from_config(c); print(n, "ctas/sm", p.info()["proj_ctas_per_sm"]); p.close()
PY
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('medium', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"
for c in large live box; do python tools/bench_live.py --config $c --reps 2 $( [ $c = large ] && echo --batch 65536 ) $( [ $c = box ] && echo --batch 16384 ) 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'ingest p50', round(d['ingest_latency_us']['p50'],1), 'readout', round(d['readout_latency_us']['p50'],1))"; done
