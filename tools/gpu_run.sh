#!/bin/bash
# Iteration run under gpurun: build, the -m gpu suite, the default bench line and a Medium line.
#   tools/gpu_run.sh <tag> [pytest -k expression]
tag=${1:-run}; kexpr=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/${tag}_build.log; exit 1; }
if [ -n "$kexpr" ]; then
  timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
else
  timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
fi
echo "pytest rc=$?"; tail -8 gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_box.json 2> gpurun_out/${tag}_bench_box.err; echo "bench rc=$?"
timeout 300 python bench.py --config medium --no-cpu-baseline --e2e-steps 3 > gpurun_out/${tag}_bench_medium.json 2> gpurun_out/${tag}_bench_medium.err; echo "bench medium rc=$?"
python - <<PY
import json
for n in ("box", "medium"):
    try:
        d = json.load(open("gpurun_out/${tag}_bench_%s.json" % n))
        print(n, "%.4g fr/s" % d["value"], "step %.3f ms" % d["ms_per_step"], "step frac %.3f" % d["step_roofline"]["frac"],
              "proj frac %.3f" % d["roofline"]["frac"], "readout us", d["latency"]["readout_us"], d["clocks"])
    except Exception as e:
        print(n, "no line", e)
PY
