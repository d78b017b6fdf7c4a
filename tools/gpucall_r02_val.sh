# full-size Graph500 validation at HEAD: s28 2x2 and s27 1x2 with the peer exchange (streaming V1-V6)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2val_build.log 2>&1
timeout 1500 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/nccl_check.py --scale 28 --roots 1 --peer --device-gen --stream-validate > gpurun_out/r2val_s28_2x2.log 2>&1; echo "rc=$?" >> gpurun_out/r2val_s28_2x2.log
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 python -m torch.distributed.run --standalone --nproc-per-node 2 tools/nccl_check.py --scale 27 --roots 1 --peer --device-gen --stream-validate > gpurun_out/r2val_s27_1x2.log 2>&1; echo "rc=$?" >> gpurun_out/r2val_s27_1x2.log
tail -2 gpurun_out/r2val_s28_2x2.log | cut -c1-500; tail -2 gpurun_out/r2val_s27_1x2.log | cut -c1-500
