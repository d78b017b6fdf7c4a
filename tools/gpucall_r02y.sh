# 2 GPUs: parent candidates pushed by K4 (no end-of-search resolution round): NCCL/peer parity tests,
# s27 1x2 peer stream-validated, 2-GPU bench (1x2, 2x1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -x -q -rs > gpurun_out/r2y2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2y2_tests.log
timeout 1200 python -m torch.distributed.run --standalone --nproc-per-node 2 tools/nccl_check.py --scale 27 --roots 2 --peer --device-gen --stream-validate > gpurun_out/r2y2_check_s27_1x2.log 2>&1; echo "rc=$?" >> gpurun_out/r2y2_check_s27_1x2.log
run() { n=$1; tag=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 20 --warmup 3 "$@" > gpurun_out/r2y2_bench_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/r2y2_bench_$tag.log; }
run 2 1x2
run 2 2x1 --grid 2x1
tail -3 gpurun_out/r2y2_tests.log; tail -8 gpurun_out/r2y2_check_s27_1x2.log
for f in gpurun_out/r2y2_bench_*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['config']['grid'], round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'], json.dumps({k: round(v,3) for k,v in d.get('phase_ms_per_step',{}).items()}))"; done
