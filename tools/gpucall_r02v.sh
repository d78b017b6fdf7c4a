# pipelined short tiles (short_tiles_p2) vs HEAD (prebuilt libheadlib.so), then GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
for rep in 1 2; do
for v in default headlib; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 --levels >> gpurun_out/r2v_ab.log 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests.log
grep -v "^  L" gpurun_out/r2v_ab.log; grep "^  L[2345]" gpurun_out/r2v_ab.log | head -10; tail -3 gpurun_out/r2v_tests.log
