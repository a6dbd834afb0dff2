python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullwdd.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for b in 512 592 444 296; do
  sed "s/kFwYBatch = 512/kFwYBatch = $b/" paper_2212_01309_b200/csrc/fullwdd.cu > /tmp/fullwdd_b.cu
  cp paper_2212_01309_b200/csrc/fullwdd.cu /tmp/fullwdd_orig.cu; cp /tmp/fullwdd_b.cu paper_2212_01309_b200/csrc/fullwdd.cu
  WDD_LIB_OUT=/tmp/libwdd_b$b.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || echo BUILD FAIL
  cp /tmp/fullwdd_orig.cu paper_2212_01309_b200/csrc/fullwdd.cu
  for c in medium large; do echo -n "batch $b: "; WDD_LIB=/tmp/libwdd_b$b.so timeout 300 python tools/bench_fullwdd.py $c | cut -c1-70; done
done
