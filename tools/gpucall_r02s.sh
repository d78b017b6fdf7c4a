# 2 GPUs: full GPU tests (incl. NCCL/peer at 2), bench 1x2 (default) and 2x1, after the resolution rewrite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/r2s_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_bench2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 3 --grid 2x1 > gpurun_out/r2s_bench2_2x1.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_bench2_2x1.log
tail -3 gpurun_out/r2s_tests.log
for f in r2s_bench2 r2s_bench2_2x1; do tail -2 gpurun_out/$f.log | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['grid'], d['value'], d['ms_per_step'], json.dumps(d['phase_ms_per_step']))"; done
