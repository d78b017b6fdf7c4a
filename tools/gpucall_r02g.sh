# 4 GPUs at HEAD: GPU tests, bench N=1 / 2 (1x2) / 4 (2x2, 4x1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g4_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2g4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g4_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2g4_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/r2g4_bench1.log
run() { n=$1; tag=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 20 --warmup 3 "$@" > gpurun_out/r2g4_bench_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/r2g4_bench_$tag.log; }
CUDA_VISIBLE_DEVICES=0,1 run 2 1x2
CUDA_VISIBLE_DEVICES=0,1 run 2 2x1 --grid 2x1
run 4 2x2
run 4 4x1 --grid 4x1
for f in gpurun_out/r2g4_bench1.log gpurun_out/r2g4_bench_*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['config']['grid'], round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'], json.dumps({k: round(v,3) for k,v in d.get('phase_ms_per_step',{}).items()}))"; done
tail -3 gpurun_out/r2g4_tests.log
