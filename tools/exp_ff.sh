#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
nproc
python - <<'PY'
import time
import paper_2212_01309_b200 as w
from synth import CONFIGS
for n in ["tiny","medium","large","live","box"]:
    c=CONFIGS[n]; t=time.time(); p=w.Plan.from_config(c); dt=time.time()-t; i=p.info(); print(n, "plan_create_s", round(dt,2), "n_act", i["n_act"], "ctas/sm", i["proj_ctas_per_sm"]); p.close()
PY
