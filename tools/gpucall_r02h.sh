# 4 GPUs: NCCL/peer parity tests, s28 2x2 peer stream-validated, 4-GPU bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r2h_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -rs > gpurun_out/r2h_nccl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_nccl_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/r2h_bench4.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_bench4.log
timeout 2400 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/nccl_check.py --scale 28 --roots 1 --peer --device-gen --stream-validate > gpurun_out/r2h_check_s28_2x2.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_check_s28_2x2.log
tail -3 gpurun_out/r2h_nccl_tests.log; tail -2 gpurun_out/r2h_bench4.log | cut -c1-400; tail -2 gpurun_out/r2h_check_s28_2x2.log | cut -c1-800
