mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/exp_tests.log
timeout 300 python tools/profile_bfs.py --roots 2 > gpurun_out/exp_p.log 2>&1
timeout 400 python bench.py > gpurun_out/exp_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/exp_bench.log
tail -2 gpurun_out/exp_tests.log; tail -10 gpurun_out/exp_p.log; tail -2 gpurun_out/exp_bench.log | cut -c1-200
