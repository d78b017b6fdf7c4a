# 1 GPU at HEAD: per-level phase times, ncu launch list, ncu --set full of the L3 launches, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 300 python tools/profile_bfs.py --roots 1 > gpurun_out/r2k_levels.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches.csv python tools/profile_bfs.py --roots 1 > gpurun_out/r2k_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_parent|k_scan_emit|k_scan_count|k_finalize" --launch-skip 12 --launch-count 5 -f -o gpurun_out/r2k_L3 python tools/profile_bfs.py --roots 1 > gpurun_out/r2k_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/r2k_L3.ncu-rep > gpurun_out/r2k_ncu_summary.txt 2>&1
cat gpurun_out/r2k_levels.log; cut -c1-250 gpurun_out/r2k_ncu_summary.txt | head -40
