# K1 RED-reuse A/B (1 GPU), then ncu captures of the default build at the peak level
mkdir -p gpurun_out
python -c "
import __graft_entry__ as g; g.build()
from paper_1408_1605_b200 import _build
_build.build_variant('k1red', ['BFS200_K1RED=1'])
" > gpurun_out/r2k_build.log 2>&1
for rep in 1 2; do
for v in default k1red; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2k_ab.log 2>&1
done; done
cat gpurun_out/r2k_ab.log
