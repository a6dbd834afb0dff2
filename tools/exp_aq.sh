#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_fullwdd.py -q 2>&1 | tail -12
for c in medium large; do timeout 300 python tools/bench_fullwdd.py $c; done
