#!/bin/bash
run() {
  for c in large live; do timeout 300 python tools/bench_live.py --config $c --reps 2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 $c', round(d['frames_per_s']/1e6,2), 'ingest p50', round(d['ingest_latency_us']['p50'],1), 'readout', round(d['readout_latency_us']['p50'],1))"; done
}
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1; run base
WDD_NVCC_EXTRA=-DWDD_EXP_NOC python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1; run noC
WDD_NVCC_EXTRA=-DWDD_EXP_NOA2 python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1; run noA2
WDD_NVCC_EXTRA="-DWDD_EXP_NOA2 -DWDD_EXP_NOC" python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1; run noboth
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
