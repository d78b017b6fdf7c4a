# A/B of the working tree against prebuilt variant libraries, then the GPU tests:
#   bash tools/gpucall_ab.sh TAG VARIANT...   (build/variants/lib<VARIANT>.so, e.g. from tools/build_rev.py)
tag=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 --levels >> gpurun_out/${tag}_ab.log 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
grep -v "^  L" gpurun_out/${tag}_ab.log; grep "^  L[12345]" gpurun_out/${tag}_ab.log | head -10; tail -3 gpurun_out/${tag}_tests.log
