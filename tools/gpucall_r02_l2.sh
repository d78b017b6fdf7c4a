# 1 GPU: ncu --set full of the level-2 (mode 3) k_expand launch at HEAD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l2_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand" --launch-skip 2 --launch-count 1 -f -o gpurun_out/r2l2_L2 python tools/profile_bfs.py --roots 1 > gpurun_out/r2l2_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2l2_L2.ncu-rep > gpurun_out/r2l2_summary.txt 2>&1
cut -c1-300 gpurun_out/r2l2_summary.txt | head -10
