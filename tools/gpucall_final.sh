mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rs > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/fin_bench1.log 2>&1; echo "bench1 rc=$?" >> gpurun_out/fin_bench1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 > gpurun_out/fin_bench2.log 2>&1; echo "bench2 rc=$?" >> gpurun_out/fin_bench2.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/fin_ref.log
tail -3 gpurun_out/fin_tests.log; tail -1 gpurun_out/fin_smoke.log; for f in fin_bench1 fin_bench2 fin_ref; do tail -2 gpurun_out/$f.log | cut -c1-160; done
