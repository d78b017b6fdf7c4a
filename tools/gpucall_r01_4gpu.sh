mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?" >> gpurun_out/bench4.log
tail -2 gpurun_out/gpu_tests4.log; tail -2 gpurun_out/bench4.log | cut -c1-300
