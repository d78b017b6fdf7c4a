# K1 deferred-RED pipeline A/B (1 GPU)
mkdir -p gpurun_out
python -c "
import __graft_entry__ as g; g.build()
from paper_1408_1605_b200 import _build
for ns in (2, 3, 4): _build.build_variant(f'pipe{ns}', [f'BFS200_K1PIPE={ns}'])
" > gpurun_out/r2e_build.log 2>&1
for v in pipe2 pipe3 pipe4; do
  BFS200_LIB=paper_1408_1605_b200/build/variants/lib$v.so timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2e_ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kron or multi_column or pos64 or s26" > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e_tests.log
cat gpurun_out/r2e_ab.log; tail -2 gpurun_out/r2e_tests.log
