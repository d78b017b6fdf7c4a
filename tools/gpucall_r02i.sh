# K1 shared-memory target A/B with the pipelined loop (1 GPU) + checked-build test
mkdir -p gpurun_out
python -c "
import __graft_entry__ as g; g.build()
from paper_1408_1605_b200 import _build
for kb in (144, 176, 192, 208): _build.build_variant(f'smem{kb}', [f'BFS200_SMEM_KB={kb}'])
_build.build_variant('checked', ['BFS200_CHECKS=1'])
" > gpurun_out/r2i_build.log 2>&1
for rep in 1 2; do
for v in default smem144 smem176 smem192 smem208; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2i_ab.log 2>&1
done; done
timeout 1200 python -m pytest tests/test_gpu_checked.py -q > gpurun_out/r2i_checked.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_checked.log
cat gpurun_out/r2i_ab.log; tail -2 gpurun_out/r2i_checked.log
