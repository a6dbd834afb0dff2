# Verification of a build (under gpurun, from the repo root): smoke, the -m gpu suite, the default bench
# line and the reference arm, the conventional-WDD comparison; outputs in gpurun_out/r02h_*.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python __graft_entry__.py smoke > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02h_smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02h_pytest.log
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02h_bench_reference.json 2>/dev/null; echo "ref rc=$?"
for c in medium large; do timeout 300 python tools/bench_fullwdd.py $c; done > gpurun_out/r02h_fullwdd.txt 2>&1
echo done
