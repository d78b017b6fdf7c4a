# round-2 evidence at HEAD (1 GPU), refresh: bench (default args), reference arm, ncu launch list and full capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r2r_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_bench1.log
timeout 900 python bench.py --impl reference --steps 16 --warmup 0 > gpurun_out/r2r_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_ref.log
export CUDA_VISIBLE_DEVICES=0
timeout 300 python tools/profile_bfs.py --roots 1 > gpurun_out/r2r_levels.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_launches.csv python tools/profile_bfs.py --roots 1 > gpurun_out/r2r_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_parent|k_scan_emit|k_scan_count|k_finalize" --launch-skip 12 --launch-count 5 -f -o gpurun_out/r2r_L3 python tools/profile_bfs.py --roots 1 > gpurun_out/r2r_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/r2r_L3.ncu-rep > gpurun_out/r2r_ncu_summary.txt 2>&1
tail -2 gpurun_out/r2r_bench1.log | cut -c1-300; tail -2 gpurun_out/r2r_ref.log | cut -c1-300; cat gpurun_out/r2r_levels.log; cut -c1-300 gpurun_out/r2r_ncu_summary.txt
