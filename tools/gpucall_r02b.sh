# round-2 GPU call B (2 GPUs): NCCL/peer parity tests, s27 1x2 peer stream-validated, 2-GPU bench, 1-GPU bench with cpu leg
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q -rs > gpurun_out/r2b_nccl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_nccl_tests.log
timeout 1200 python -m torch.distributed.run --standalone --nproc-per-node 2 tools/nccl_check.py --scale 27 --roots 2 --peer --device-gen --stream-validate > gpurun_out/r2b_check_s27_1x2.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_check_s27_1x2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/r2b_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_bench2.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/r2b_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_bench1.log
tail -3 gpurun_out/r2b_nccl_tests.log; tail -2 gpurun_out/r2b_check_s27_1x2.log | cut -c1-600; tail -2 gpurun_out/r2b_bench2.log | cut -c1-300; tail -2 gpurun_out/r2b_bench1.log | cut -c1-300
