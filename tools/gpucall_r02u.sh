# 4 GPUs: GPU tests (NCCL/peer at 2 and 4), bench 2x2 (default) and 4x1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/r2u_bench4.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --steps 20 --warmup 3 --grid 4x1 > gpurun_out/r2u_bench4_4x1.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench4_4x1.log
tail -3 gpurun_out/r2u_tests.log
for f in r2u_bench4 r2u_bench4_4x1; do tail -2 gpurun_out/$f.log | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['grid'], d['value'], d['ms_per_step'], json.dumps(d['phase_ms_per_step']))"; done
