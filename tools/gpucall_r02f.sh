# K1 pipe A/B, full GPU tests (incl. SNAP), compute-sanitizer runs (1 GPU)
mkdir -p gpurun_out/sanitizer
python -c "
import __graft_entry__ as g; g.build()
from paper_1408_1605_b200 import _build
for ns in (2, 4): _build.build_variant(f'pipe{ns}', [f'BFS200_K1PIPE={ns}'])
" > gpurun_out/r2f_build.log 2>&1
for v in default pipe2 pipe4; do
  if [ $v = default ]; then L=""; else L=paper_1408_1605_b200/build/variants/lib$v.so; fi
  BFS200_LIB=$L timeout 300 python tools/ab_expand.py --roots 8 >> gpurun_out/r2f_ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f_tests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer/r02_${tool}_s12.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/r02_${tool}_s12.log
done
SAN_SCALE=18 timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer/r02_racecheck_s18.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/r02_racecheck_s18.log
SAN_SCALE=18 timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer/r02_memcheck_s18.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/r02_memcheck_s18.log
cat gpurun_out/r2f_ab.log; tail -3 gpurun_out/r2f_tests.log; for f in gpurun_out/sanitizer/r02_*; do echo $f; tail -3 $f; done
