# new K3 CTA-level scan timing + ncu captures at the peak level (1 GPU)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 300 python tools/ab_expand.py --roots 8 --levels > gpurun_out/r2d_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_tests.log
export CUDA_VISIBLE_DEVICES=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_parent|k_scan_emit|k_scan_count" --launch-skip 12 --launch-count 4 -f -o gpurun_out/r2d_L3 python tools/profile_bfs.py --roots 1 > gpurun_out/r2d_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2d_L3.ncu-rep > gpurun_out/r2d_ncu_summary.txt 2>&1
cat gpurun_out/r2d_ab.log | grep -v "^  L[5-9]"; tail -2 gpurun_out/r2d_tests.log; cat gpurun_out/r2d_ncu_summary.txt | cut -c1-400
