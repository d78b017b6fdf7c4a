# K1 long-tile variant A/B, interleaved x2 (1 GPU)
mkdir -p gpurun_out
python -c "
import __graft_entry__ as g; g.build()
from paper_1408_1605_b200 import _build
for v in (0,1,2): _build.build_variant(f'k1v{v}', [f'BFS200_K1VAR={v}'])
_build.build_variant('pipe0', ['BFS200_K1PIPE=0'])
" > gpurun_out/r2g_build.log 2>&1
for rep in 1 2; do
for v in k1v0 k1v1 k1v2 pipe0; do
  BFS200_LIB=paper_1408_1605_b200/build/variants/lib$v.so timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2g_ab.log 2>&1
done; done
cat gpurun_out/r2g_ab.log
