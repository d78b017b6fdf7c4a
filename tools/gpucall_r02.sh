# round-2 GPU call: tests, smoke, short bench (1 GPU)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_box.txt 2>&1
nproc >> gpurun_out/r2_box.txt; free -g >> gpurun_out/r2_box.txt; lscpu | grep -i "model name" >> gpurun_out/r2_box.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench1.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench1.log
tail -4 gpurun_out/r2_tests.log; tail -1 gpurun_out/r2_smoke.log; tail -2 gpurun_out/r2_bench1.log | cut -c1-300
