# single visited bitmap (vis/vold) vs the interleaved pair layout (prebuilt libpairs.so), 1 GPU
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
for rep in 1 2; do
for v in default pairs; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2j_ab.log 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
cat gpurun_out/r2j_ab.log; tail -3 gpurun_out/r2j_tests.log
