mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?" >> gpurun_out/bench2.log
export CUDA_VISIBLE_DEVICES=0
timeout 300 python tools/profile_bfs.py --roots 1 > gpurun_out/p.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_bfs.py --roots 1 > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expand --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_expand_L3 python tools/profile_bfs.py --roots 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/gpu_tests2.log; tail -2 gpurun_out/bench2.log | cut -c1-400; tail -12 gpurun_out/p.log; tail -3 gpurun_out/ncu_full.log
