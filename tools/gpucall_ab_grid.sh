# A/B on a loopback grid (all ranks on one GPU): bash tools/gpucall_ab_grid.sh TAG GRID SCALE VARIANT...
tag=$1; grid=$2; scale=$3; shift 3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 400 python tools/ab_expand.py --roots 8 --grid $grid --scale $scale >> gpurun_out/${tag}_ab.log 2>&1
done; done
grep -v "^  L" gpurun_out/${tag}_ab.log
