# 1 GPU: bfs_run_batch (pipelined host copies): its parity test, the GPU suite, bench N=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2bt_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k run_batch > gpurun_out/r2bt_batch.log 2>&1; echo "rc=$?" >> gpurun_out/r2bt_batch.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2bt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2bt_tests.log
timeout 900 python bench.py > gpurun_out/r2bt_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/r2bt_bench1.log
tail -3 gpurun_out/r2bt_batch.log; tail -3 gpurun_out/r2bt_tests.log
grep '^{' gpurun_out/r2bt_bench1.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e']))"
