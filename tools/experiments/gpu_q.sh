#!/bin/bash
# quick iteration: build + selected gpu tests (+ optional extra command)
tag=$1; kexpr=$2; extra=$3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/${tag}_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error|error" gpurun_out/${tag}_pytest.log | tail -15
if [ -n "$extra" ]; then bash -c "$extra"; fi
